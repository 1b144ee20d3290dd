"""Per-step cost of the partition exchange on one GPU: C4 as one
partition, and as 8 partitions in one process with the copy transport
(migration regions + k_absorb + halo pack / copy / unpack) and with the direct
transport (NEXT-2: k_step stores movers and summaries into the owner's
buffers; nothing after the step).  The 8-partition runs do the same
vehicle-steps as the single partition, so the difference is the exchange."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2406_10661_b200 as p

scen = synth.city()                       # (not the npz cache: the partitioner needs the geometry)
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
own = synth.rcb_partition(scen, W)
out = {"workload": "C4", "partitions": W}
PRE = int(os.environ.get("PREROLL", "200"))
out["preroll_steps"] = PRE
out["note"] = "sim_step(40) timed with CUDA events: step graphs (6 steps per replay, PDL) unless *_eager"
for name, kw in (("single", {}), ("single_eager", dict(step_graphs=False)),
                 ("copy", dict(world=W, loopback=True, road_owner=own)),
                 ("direct", dict(world=W, loopback=True, direct=True, road_owner=own)),
                 ("direct_eager", dict(world=W, loopback=True, direct=True, road_owner=own,
                                       step_graphs=False))):
    st = torch.cuda.Stream()
    sim = p.Sim.from_scenario(scen, stream=st.cuda_stream, **kw)
    sim.step(PRE)
    sim.sync()
    m0 = sim.read_metrics()
    n = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        sim.step(n)
        e1.record(st)
    torch.cuda.synchronize()
    m1 = sim.read_metrics()
    ms = e0.elapsed_time(e1) / n
    out[name] = {"ms_per_step": ms, "vehicle_steps_per_s": (m1["vehicle_steps"] - m0["vehicle_steps"]) / (ms * n / 1e3)}
    del sim
    torch.cuda.synchronize()
print(json.dumps(out))
