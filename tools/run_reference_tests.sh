#!/bin/bash
# The reference's own test files against the GPU backend (run under gpurun).
# Needs the reference staged under baseline/_ref (git-ignored, travels with
# the snapshot): pip install --no-index --no-deps --target baseline/_ref
# <copy of /root/reference/pkg>, plus its tests copied to baseline/_ref/ref_tests.
# The plugin swaps mdtune's ForceCalculator for HostForceCalculator in
# pytest_configure, before the test modules bind the name.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$(realpath -m "${1:-$ROOT/gpurun_out/ref_tests.log}")
mkdir -p "$(dirname "$OUT")"
cd "$ROOT/baseline/_ref/ref_tests"
export PYTHONPATH="$ROOT/baseline/_ref:$ROOT"
export NUMBA_CACHE_DIR=/tmp/mdg_numba_cache
python -m pytest -p paper_2505_03438_b200.plugin -p no:cacheprovider --rootdir . -rA \
    test_containers.py test_simulation.py test_integrator.py test_dataset.py \
    test_cells.py test_forces.py test_configuration.py test_livestats.py test_tuning.py \
    test_fuzzy.py test_forest.py test_rules.py test_scenarios.py test_experiments.py \
    "test_acceptance.py::test_criterion_1_forces_match_oracle_on_random_scenarios" \
    "test_acceptance.py::test_criterion_2_search_space_has_exactly_the_valid_30" \
    "test_acceptance.py::test_criterion_3_c08_directed_interactions_halve_under_newton3" \
    > "$OUT" 2>&1
rc=$?
tail -5 "$OUT"
exit $rc
