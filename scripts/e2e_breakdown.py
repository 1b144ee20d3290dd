"""Time the pieces of the bench e2e loop on C4 (dev tool)."""
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
ph = np.zeros(nj, np.int32)
def t(f, n=20):
    sim.sync(); t0 = time.perf_counter()
    for _ in range(n): f()
    sim.sync(); return (time.perf_counter() - t0) / n * 1e3
print("step only        %.3f ms" % t(lambda: sim.step(1)))
print("set_phase_batch  %.3f ms" % t(lambda: sim.set_signal_phase_batch(jids, ph)))
print("read_metrics     %.3f ms" % t(lambda: sim.read_metrics()))
print("read_metrics+ln  %.3f ms" % t(lambda: sim.read_metrics(lane_stats=True)))
def loop():
    sim.set_signal_phase_batch(jids, ph); sim.step(1); sim.read_metrics(lane_stats=True)
print("e2e loop         %.3f ms" % t(loop))
