"""Time the pieces of the bench e2e loop on C4 (dev tool): host time of each
call of one RL-style step (controller, set_signal_phase_batch, sim_step,
read_metrics with lane statistics, which synchronises)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2406_10661_b200.sim as S
cache = "/tmp/c4.npz"
scen = synth.load_scenario(cache) if os.path.exists(cache) else synth.city()
if not os.path.exists(cache):
    synth.save_scenario(scen, cache)
st = torch.cuda.Stream()
sim = S.Sim.from_scenario(scen, stream=st.cuda_stream)
sim.step(5); sim.sync()
nj = len(scen.graph["junc_lane_offsets"]) - 1
jids = np.arange(nj, dtype=np.int32)
offs = scen.graph["junc_offset_steps"].astype(np.int64)
tau_phase = np.where(np.arange(102) < 33, 0, np.where(np.arange(102) < 51, 1,
                     np.where(np.arange(102) < 84, 2, 3))).astype(np.int32)
plan = np.ascontiguousarray(tau_phase[(np.arange(102)[:, None] + offs[None, :]) % 102])
obs_buf = {k: torch.empty(scen.n_lanes, dtype=torch.int32, pin_memory=True).numpy()
           for k in ("lane_count", "lane_waiting_at_end")}
acc = np.zeros(5)
n = 50
m0 = sim.read_metrics()
for k in range(n):
    t0 = time.perf_counter()
    ph = plan[(m0["t"] + k) % 102]
    t1 = time.perf_counter()
    sim.set_signal_phase_batch(jids, ph)
    t2 = time.perf_counter()
    sim.step(1)
    t3 = time.perf_counter()
    obs = sim.read_metrics(lane_stats=True, out=obs_buf)
    t4 = time.perf_counter()
    acc += [t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0]
acc = acc / n * 1e3
print("controller %.3f  set_phase %.3f  step(launch) %.3f  read_metrics+lanes(sync) %.3f  total %.3f ms" % tuple(acc))
