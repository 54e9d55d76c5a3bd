"""Host drift / kick throughput of libmdg's native integrator on pinned
arrays (the e2e path's host passes), 1,048,576 particles, both layouts."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import hostloop  # noqa: E402

n = 1_048_576
L = 111.8183
rng = np.random.default_rng(0)
params = P.SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3, boundary=(P.PERIODIC,) * 3)
for layout in ("AoS", "SoA"):
    p = hostloop.HostParticleSet(rng.uniform(0, L, (n, 3)), rng.normal(0, 1, (n, 3)), layout=layout)
    p.force[:] = rng.normal(0, 1, p.force.shape)
    for name, fn in (("drift", lambda: hostloop.host_drift_wrap(p, params, 1e-3)),
                     ("kick", lambda: hostloop.host_finish_kick(p, 1e-3))):
        fn()
        best = 1e9
        for _ in range(10):
            t = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t)
        mb = (144 if name == "drift" else 96) * n / 1e6
        print(f"{layout} {name}: {best * 1e3:.3f} ms  ({mb / best / 1e3:.0f} GB/s of {mb:.0f} MB nominal)")
