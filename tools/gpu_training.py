"""GPU-labelled training data, forest and rule file.

Runs the reference's own training roster (mdtune.dataset.dataset_scenarios,
dataset.py:200-260: uniform fills, Gaussian clusters, hex slabs in a gas,
lattice spheres, an empty box; skins 0.1-0.5 x thread counts 1/2/4/8) with
every configuration trialled on the DEVICE (paper_2505_03438_b200.dataset:
CUDA-event timings, device live statistics), writes the reference's CSV
layout, trains the forest with the reference's own trainer
(dataset.py:230-235 train_forest_from_csv, forest.py:262-269 save_forest) and
distils a rule file in the reference's format (data/default_rules.txt) from
the same sweep.

The reference package is needed (its roster, scenario generators and
trainer): it is the staged, unmodified install under baseline/_ref.

    python tools/gpu_training.py [--out paper_2505_03438_b200/data]

Outputs: gpu_training.csv, gpu_forest.json, gpu_rules.txt (+ a summary).
The tuning space is the reference's 30 ids plus the exact GPU-only
Verlet-cluster-list ids (the fp32 variant is a precision choice, not a
performance knob, and stays out).
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF):
    sys.path.append(REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mdg_numba_cache")

import numpy as np  # noqa: E402

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import dataset  # noqa: E402
from paper_2505_03438_b200.configuration import tuning_space  # noqa: E402


def roster_points(scale, cap):
    """(our ParticleSet, our SimulationParams) for every sweep point of the
    reference roster, in the reference's order (dataset.py:149-202)."""
    from mdtune.dataset import DATASET_SKINS, DESK_THREADS, dataset_scenarios
    from mdtune.scenarios import generate_scenario
    for spec in dataset_scenarios(scale, cap):
        try:
            base = generate_scenario(spec)
        except Exception as exc:   # the reference logs and skips these too
            print(f"scenario {spec.name} failed to generate: {exc}", file=sys.stderr)
            continue
        types = [P.ParticleTypeInfo(t.type_id, t.epsilon, t.sigma, t.mass) for t in base.types]
        for skin in DATASET_SKINS:
            for threads in DESK_THREADS:
                params = P.SimulationParams(domain_size=spec.params.domain_size,
                                            cutoff=spec.params.cutoff, skin=skin,
                                            rebuild_interval=spec.params.rebuild_interval,
                                            boundary=spec.params.boundary, thread_count=threads)
                parts = P.ParticleSet(np.asarray(base.positions), np.asarray(base.velocities),
                                      type_ids=np.asarray(base.type_id), types=types)
                yield spec.name, parts, params


TERMS = (("Sparse", "trap 0 0 4 10"), ("Moderate", "trap 4 10 48 96"), ("Dense", "trap 48 96 256 256"))


def _term_of(max_per_bin):
    return "Sparse" if max_per_bin < 7 else "Moderate" if max_per_bin < 72 else "Dense"


def distil_rules(csv_path, space_ids, top=3):
    """A rule file in the reference's grammar (fuzzy.py:283-380) from the GPU
    sweep: maxParticlesPerBin, the input the reference's own rules key on,
    split into the same three terms; per term the configurations that win
    (lowest device cost) most often -- and those within 10% of the winner --
    are Good there, every other configuration Bad."""
    import csv
    with open(csv_path) as fh:
        rows = list(csv.DictReader(fh))
    good = {t: collections.Counter() for t, _ in TERMS}
    for r in rows:
        term = _term_of(float(r["maxParticlesPerBin"]))
        costs = {c: float(r[f"cost:{c}"]) for c in space_ids}
        best = min(costs.values())
        for c, v in costs.items():
            if v <= 1.1 * best:
                good[term][c] += 1
    chosen = {t: [c for c, _ in good[t].most_common(top)] for t in good}
    out = ["# GPU selector rules, distilled from the device-timed sweep of the",
           "# reference's training roster (tools/gpu_training.py): per bin-occupancy",
           "# term, the configurations within 10% of the fastest most often.", "",
           "var maxParticlesPerBin 0 256",
           "term maxParticlesPerBin.Any trap 0 0 256 256"]
    out += [f"term maxParticlesPerBin.{t} {shape}" for t, shape in TERMS]
    out.append("")
    for cid in space_ids:
        terms = [t for t in good if cid in chosen[t]]
        if terms:
            cond = " or ".join(f"maxParticlesPerBin == {t}" for t in terms)
            out.append(f'rule if {cond} then "{cid}".Suitability == Good')
            out.append(f'rule if not ({cond}) then "{cid}".Suitability == Bad')
        else:
            out.append(f'rule if maxParticlesPerBin == Any then "{cid}".Suitability == Bad')
    return "\n".join(out) + "\n", chosen


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2505_03438_b200", "data"))
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("--cap", type=int, default=10_000)
    ap.add_argument("--trials", type=int, default=dataset.TRIAL_ITERATIONS)
    a = ap.parse_args()
    from mdtune.dataset import train_forest_from_csv
    from mdtune.forest import save_forest
    from mdtune.fuzzy import parse_rule_file
    os.makedirs(a.out, exist_ok=True)
    space = tuning_space()
    ids = [c.id for c in space]
    csv_path = os.path.join(a.out, "gpu_training.csv")
    labels = collections.Counter()
    points = ((p, prm) for _, p, prm in roster_points(a.scale, a.cap))
    rows = dataset.generate_training_dataset(csv_path, points, space=space, trial_iterations=a.trials,
                                             progress=lambda k, lab: labels.update([lab]))
    forest = train_forest_from_csv(csv_path, n_estimators=100, seed=0)
    save_forest(forest, os.path.join(a.out, "gpu_forest.json"))
    text, chosen = distil_rules(csv_path, ids)
    parse_rule_file(text, space)     # the reference's parser accepts it
    with open(os.path.join(a.out, "gpu_rules.txt"), "w") as fh:
        fh.write(text)
    summary = {"rows": rows, "labels": dict(labels.most_common()), "good_by_term": chosen,
               "forest_classes": list(forest.classes)}
    with open(os.path.join(a.out, "gpu_training_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
