"""SURVEY §8(d) supporting numbers on the box (one B200):
  * fixed-cost floor of a step: sim_step(1) on C1 (1 km ring, 20 vehicles),
    device time per step with CUDA events — launches + the persistent step
    kernel's minimum, no bandwidth;
  * L2-resident copy bandwidth (24 MiB -> 24 MiB, repeated) next to the HBM copy
    peak of MEASURED_PEAKS.json, to place the 2M-vehicle working set;
  * the issue ceiling used for the k_step issue fraction: 148 SMs x 4 warp
    schedulers x 1 warp-instruction / cycle at the max SM clock.
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2406_10661_b200 as p

out = {}
scen = synth.ring()
st = torch.cuda.Stream()
sim = p.Sim.from_scenario(scen, stream=st.cuda_stream)
sim.step(20)
sim.sync()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
sim.step(n)
e1.record(st)
torch.cuda.synchronize()
out["c1_step_floor_us"] = e0.elapsed_time(e1) / n * 1e3
a = torch.empty(24 << 20, dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
for _ in range(10):
    b.copy_(a)
torch.cuda.synchronize()
reps = 200
e0.record()
for _ in range(reps):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
out["l2_copy_gbs"] = 2 * a.numel() * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
prop = torch.cuda.get_device_properties(0)
out["sm_count"] = prop.multi_processor_count
out["l2_bytes"] = getattr(prop, "L2_cache_size", None)
try:
    mp = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    out["hbm_copy_gbs_measured"] = mp.get("hbm_gbs")
    clk = mp.get("sm_max_mhz", 1965.0)
except Exception:
    clk = 1965.0
out["issue_peak_warp_inst_per_s"] = prop.multi_processor_count * 4 * clk * 1e6
print(json.dumps(out))
