"""Full-run aggregates of the oracle (VERDICT r01 "Next round" #2c/#2d).

tests/golden/oracle_aggregates.json was written by scripts/oracle_aggregates.py,
which calls only oracle/.  Here (no GPU):
  * the stored C2 values are reproduced by the oracle (a regression pin of the
    stored file: it came from this oracle, not from the CUDA path);
  * the scatter of the oracle against itself with fp32 state storage (the
    storage precision of the GPU path) is measured per seed.  In
    this congested scenario the dynamics are chaotic: rounding the state to
    fp32 moves ATT / mean wait by more than north_star's 0.5% on a single
    seed, so a per-run 0.5% bar cannot be met by ANY fp32-storage
    implementation, including the oracle itself.  The GPU tests therefore
    compare exact mode (fp64 arithmetic, fp32 storage) with the stored
    fp32-storage values exactly, per run, and the fp32 path pooled over seeds
    (DESIGN §4.3).
"""
import json
import os

import pytest

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_aggregates.json")))
KEYS = ("tp", "att_finished", "att_all", "mean_wait", "vehicle_steps", "n_driving")


def _agg(m):
    nf = m["n_finished"]
    return dict(tp=nf, att_finished=m["att_finished"], att_all=m["att_all"],
                mean_wait=m["sum_wait_steps_finished"] / nf, vehicle_steps=m["vehicle_steps"],
                n_driving=m["n_driving"])


@pytest.mark.parametrize("seed", [2, 3])
def test_stored_c2_aggregates_reproduce(oracle_lib, seed):
    scen = synth.grid(seed=seed)
    for mode, fp32 in (("fp64", False), ("fp32store", True)):
        o = oracle_lib.Oracle(scen, store_fp32=fp32)
        o.step(3600)
        got = _agg(o.metrics())
        want = GOLD[f"C2-seed{seed}-{mode}"]
        for k in KEYS:
            assert got[k] == pytest.approx(want[k], rel=1e-12), (seed, mode, k)


def test_fp32_storage_scatter_exceeds_half_percent():
    """The oracle's own fp64 vs fp32-storage runs differ by more than 0.5% in
    ATT or mean wait on at least one C2 seed (the measured reason for the
    pooled fp32 comparison)."""
    worst = 0.0
    for seed in (2, 3):
        a, b = GOLD[f"C2-seed{seed}-fp64"], GOLD[f"C2-seed{seed}-fp32store"]
        for k in ("att_finished", "mean_wait"):
            worst = max(worst, abs(a[k] - b[k]) / abs(a[k]))
    assert worst > 0.005, worst
