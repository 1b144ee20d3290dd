"""Batched environments (NEXT-3) throughput: B independent C2 environments
(4x4 signalised grid, 2-lane roads, 5k trips, fixed-time signals; each its
own seed) stepped by one sim_step.  Warm-up W steps from t = 0 (departures
fill the networks), then K timed steps with CUDA events on the sim stream.
Prints one JSON line (vehicle-steps/s and environment-steps/s)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2406_10661_b200 as p

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=256)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--warmup", type=int, default=900)
a = ap.parse_args()
t0 = time.time()
envs = [synth.grid(seed=1000 + e) for e in range(a.envs)]
B = synth.batch(envs)
gen_s = time.time() - t0
st = torch.cuda.Stream()
sim = p.Sim.from_scenario(B, stream=st.cuda_stream)
sim.step(a.warmup)
m0 = sim.read_metrics()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
sim.step(a.steps)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
m1 = sim.read_metrics()
gm = sim.read_group_metrics(a.envs)
vs = m1["vehicle_steps"] - m0["vehicle_steps"]
print(json.dumps({
    "metric": "vehicle-steps/sec", "value": vs / (ms / 1e3), "unit": "vehicle-steps/s",
    "env_steps_per_s": a.envs * a.steps / (ms / 1e3), "ms_per_step": ms / a.steps,
    "config": {"workload": f"{a.envs} batched C2 environments (4x4 grid, 2 lanes, 5k trips each, "
                           f"fixed time, seeds 1000..), steps {a.warmup}..{a.warmup + a.steps}",
               "n_lanes": int(B.n_lanes), "n_trips": int(B.n_trips),
               "driving_mean": vs / a.steps, "generation_s": round(gen_s, 1)},
    "finished_per_env_mean": float(np.mean([g["n_finished"] for g in gm])),
    "note": "no L2 flush between steps; total state fits L2"}))
