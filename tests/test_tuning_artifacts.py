"""the GPU-labelled training CSV, forest and rule file
(paper_2505_03438_b200/data, written by tools/gpu_training.py on a B200 from
the reference's own roster and trainer) load through the reference's own
readers, and its Expert / Random-Forest strategies then propose the
configurations the GPU measured fastest -- including the GPU-only
Verlet-cluster-list ids -- where the shipped CPU rules propose cell
traversals.  CPU-only: needs the reference package (staged under
baseline/_ref, or the read-only tree in the build container)."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import port

for _p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(_p, "mdtune")) and _p not in sys.path:
        sys.path.append(_p)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mdg_numba_cache")
mdtune = pytest.importorskip("mdtune", reason="reference package not available")

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import dataset  # noqa: E402


class _Stats:
    def __init__(self, fv):
        self.fv = np.asarray(fv, dtype=np.float64)

    def feature_vector(self):
        return self.fv


def _stats(n, side, threads=8, skin=0.3, seed=0):
    rng = np.random.default_rng(seed)
    p = port.Particles(rng.uniform(0.0, side, (n, 3)))
    params = port.Params(domain_size=(side,) * 3, cutoff=3.0, skin=skin,
                         boundary=(port.PERIODIC,) * 3, thread_count=threads)
    return _Stats(port.compute_live_stats(p, params))


GPU_IDS = {"VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS", "VCL-ClusterIter-NoN3L-SoA",
           "VCL-ClusterIter-NoN3L-AoS", "VCL-ClusterIter-N3L-SoA", "VCL-ClusterIter-N3L-AoS"}


def test_training_csv_reads_with_the_reference_loader():
    from mdtune.dataset import load_training_csv
    feats, labels = load_training_csv(dataset.GPU_TRAINING_CSV)
    space = {c.id for c in P.tuning_space()}
    assert feats.shape == (len(labels), 8) and len(labels) >= 500
    assert set(labels) <= space
    assert any(lab.startswith("VCL-") for lab in labels)   # GPU-only ids win some points
    with open(os.path.join(dataset.DATA_DIR, "gpu_training_summary.json")) as fh:
        assert json.load(fh)["rows"] == len(labels)


def test_random_forest_strategy_proposes_gpu_configurations():
    from mdtune.forest import RandomForestStrategy, rf_candidates
    forest = dataset.load_gpu_forest()
    space = P.tuning_space()
    for n, side in ((8000, 22.0), (500, 20.0), (6000, 17.0)):
        cands = rf_candidates(_stats(n, side), forest, space, k=3)
        assert cands and all(c in space for c in cands)
        assert cands[0].id in GPU_IDS, (n, side, [c.id for c in cands])
    # through the strategy object the controller calls (tuning.py:248-260)
    st = RandomForestStrategy(forest)
    assert st.candidates(space, 0, {}, _stats(8000, 22.0), None)[0].id in GPU_IDS


def test_expert_strategy_with_gpu_rules_proposes_gpu_configurations():
    from mdtune.fuzzy import ExpertStrategy, expert_candidates, parse_rule_file
    from mdtune.rules import default_rule_base
    space = P.tuning_space()
    rb = parse_rule_file(dataset.gpu_rules_text(), space)
    dense = _stats(8000, 22.0)
    got = {c.id for c in expert_candidates(dense, rb, space)}
    assert got and got <= GPU_IDS
    assert {c.id for c in ExpertStrategy(rb).candidates(space, 0, {}, dense, None)} == got
    # the shipped (CPU-trained) rules pick cell traversals for the same scene
    cpu = {c.id for c in expert_candidates(dense, default_rule_base(P.enumerate_configurations()),
                                           P.enumerate_configurations())}
    assert any(cid.startswith("LC-") for cid in cpu)
