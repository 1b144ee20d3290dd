"""Full-run aggregates of the CPU oracle (VERDICT r01 "Next round" #2c/#2d).

Runs ONLY oracle/ (no CUDA path) and writes tests/golden/oracle_aggregates.json:
  * C2 (synth.grid defaults: 4x4 signalised grid, 2 lanes, 5k trips, fixed
    time) for demand seeds 2 and 3, 3600 steps, in fp64 and with fp32 state
    storage (store_fp32, the GPU's storage precision);
  * C3 (20x20 grid, 3 lanes + tidal centre lane + dynamic middle lane, 200k
    trips, seed 3) for 3600 steps with a state-independent lane controller
    (dynamic lanes flip every 30 steps, tidal lanes every 60).
Aggregates: TP = finished trips, ATT over finished trips and over
all vehicles, mean waiting steps of finished trips,
vehicle-steps.

    python scripts/oracle_aggregates.py [--only c2|c3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_aggregates.json")
STEPS = 3600


def c3_scenario():
    return synth.grid(rows=20, cols=20, road_len=500.0, lanes=3, n_trips=200_000,
                      depart_window=1200, seed=3, tidal=True, dynamic=True)


def c3_controller(scen):
    """(t, lanes, dirs) setter calls of the fixed controller, applied before step t."""
    kinds = scen.graph["lane_kind"]
    dyn = np.where(kinds == 1)[0]
    tid = np.where((kinds == 2) & (scen.graph["tidal_partner"] > np.arange(scen.n_lanes)))[0]
    calls = []
    for t in range(0, STEPS, 30):
        calls.append((t, dyn, np.full(len(dyn), (t // 30) % 2, np.int32)))
        if t % 60 == 0:
            calls.append((t, tid, np.full(len(tid), (t // 60) % 2, np.int32)))
    return calls


def aggregates(m):
    nf = m["n_finished"]
    return dict(tp=int(nf), att_finished=float(m["att_finished"]), att_all=float(m["att_all"]),
                mean_wait=float(m["sum_wait_steps_finished"] / nf) if nf else 0.0,
                vehicle_steps=int(m["vehicle_steps"]), n_driving=int(m["n_driving"]))


def run(scen, store_fp32=False, controller=None):
    o = oracle.Oracle(scen, store_fp32=store_fp32)
    calls = {}
    for t, lanes, dirs in (controller or []):
        calls.setdefault(t, []).append((lanes, dirs))
    t = 0
    while t < STEPS:
        for lanes, dirs in calls.get(t, []):
            for l, d in zip(lanes, dirs):
                o.set_lane_direction(int(l), int(d))
        nxt = min([x for x in calls if x > t] + [STEPS])
        o.step(nxt - t)
        t = nxt
    return aggregates(o.metrics())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["c2", "c3"])
    a = ap.parse_args()
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    res["_about"] = ("Written by scripts/oracle_aggregates.py (oracle/ only). Full-run aggregates, "
                     f"{STEPS} steps: TP (finished trips, P:880-883), ATT over finished trips "
                     "(P:875-878) and over all vehicles (P:876, ledger L27), mean waiting steps of "
                     "finished trips (P:863), vehicle-steps. fp64 = the oracle as is; fp32store = "
                     "positions / speeds rounded to fp32 after every step (DESIGN 1.8).")
    if a.only in (None, "c2"):
        for seed in (2, 3):
            scen = synth.grid(seed=seed)
            for mode, fp32 in (("fp64", False), ("fp32store", True)):
                t0 = time.time()
                res[f"C2-seed{seed}-{mode}"] = run(scen, store_fp32=fp32)
                print(f"C2 seed {seed} {mode}: {res[f'C2-seed{seed}-{mode}']} ({time.time() - t0:.0f} s)", flush=True)
        json.dump(res, open(OUT, "w"), indent=1)
    if a.only in (None, "c3"):
        scen = c3_scenario()
        for mode, fp32 in (("fp64", False), ("fp32store", True)):
            t0 = time.time()
            res[f"C3-seed3-{mode}"] = run(scen, store_fp32=fp32, controller=c3_controller(scen))
            print(f"C3 {mode}: {res[f'C3-seed3-{mode}']} ({time.time() - t0:.0f} s)", flush=True)
            json.dump(res, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
