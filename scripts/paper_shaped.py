"""Context run (SURVEY §8(d) "C4-paper-shaped"; not a BASELINE config): a
network and demand shaped like the paper's largest performance dataset,
Roadnet-L (93,564 roads, 26,479 junctions, 2,464,950 vehicles, 3600 steps;
PAPER.md table tab:perf_stat), simulated for 3600 steps as in P:897.
The paper reports 42.81 s for Roadnet-L (84.09 Hz) on an RTX
4090 — different hardware and network, quoted as context only.

Network: the C4 city recipe at G = 163 with 300 m spacing (about 95k roads,
26.6k junctions).  Demand: 2,464,950 trips with 20-road biased random-walk
routes, departing uniformly over [0, 3600) s from their (non-overlapping)
start positions (P:300-305 shape).  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_2406_10661_b200 as p

t0 = time.time()
scen = synth.city(G=163, spacing=300.0, n_vehicles=2_464_950, seed=6, route_len=20)
n = scen.n_trips
rng = np.random.default_rng(6)
scen.trips["on_network_at_t0"] = np.zeros(n, np.uint8)
scen.trips["depart_step"] = rng.integers(0, 3600, n).astype(np.int32)
gen_s = time.time() - t0
st = torch.cuda.Stream()
sim = p.Sim.from_scenario(scen, stream=st.cuda_stream)
sim.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter()
e0.record(st)
sim.step(3600)
e1.record(st)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
dev_s = e0.elapsed_time(e1) / 1e3
m = sim.read_metrics()
out = {"workload": "paper-shaped context run: C4 recipe at G=163, 300 m spacing, "
                   f"{len(scen.graph['road_lane_offsets']) - 1} roads, "
                   f"{len(scen.graph['junc_lane_offsets']) - 1} junctions, {scen.n_lanes} lanes, "
                   f"{n} trips departing U[0, 3600) s, 20-road random-walk routes",
       "steps": 3600, "device_s": dev_s, "wall_s": wall, "steps_per_s": 3600 / dev_s,
       "vehicle_steps": m["vehicle_steps"], "vehicle_steps_per_s": m["vehicle_steps"] / dev_s,
       "finished": m["n_finished"], "driving_at_end": m["n_driving"],
       "pending_at_end": m["n_pending"], "att_finished_s": m["att_finished"],
       "generation_s": gen_s,
       "paper_context": {"dataset": "Roadnet-L (93,564 roads, 26,479 junctions, 2,464,950 vehicles)",
                         "seconds_3600_steps": 42.81, "hz": 84.09,
                         "hardware": "RTX 4090 + Xeon 8462Y", "cite": "P:238, P:244, P:899, P:1155",
                         "note": "different hardware and network: context, not a target"}}
print(json.dumps(out), flush=True)
