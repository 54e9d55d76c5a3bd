"""Small VL repro on a golden system (debug aid): python tools/repro_vl.py [name] [config]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200.calculator import compute_forces  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "crit1_0"
cid = sys.argv[2] if len(sys.argv) > 2 else "VL-List_Iter-NoN3L-AoS"
d = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"sys_{name}.npz"))
nt = int(d["n_types"])
types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(nt)]
per = tuple(P.PERIODIC if f else P.REFLECTIVE for f in d["periodic"])
params = P.SimulationParams(domain_size=d["domain"], cutoff=float(d["cutoff"]), skin=float(d["skin"]),
                            boundary=per)
parts = P.ParticleSet(d["pos"], type_ids=d["tid"], types=types)
cfg = P.parse_configuration(cid)
_, count = compute_forces(parts, cfg, params)
k = [str(s) for s in d["config_ids"]].index(cid)
err = np.linalg.norm(parts.numpy("force") - d["forces"][k]) / np.linalg.norm(d["forces"][k])
print(name, cid, "count", count, "ref", int(d["counts"][k]), "rel err", err)
