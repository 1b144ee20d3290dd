"""Finish-time spread of k_step_w's CTAs on C4 (dev tool; KW_TAIL builds):
how long the first CTAs idle while the last ones finish."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2406_10661_b200.sim as S
lib = sys.argv[1]
scen = synth.load_scenario("/tmp/c4.npz") if os.path.exists("/tmp/c4.npz") else synth.city()
L = S.load_library(lib)
st = torch.cuda.Stream()
sim = S.Sim.from_scenario(scen, stream=st.cuda_stream)
sim.step(200); sim.sync()
buf = (ctypes.c_ulonglong * 4096)()
spreads = []
for k in range(5):
    sim.step(1); sim.sync()
    if L.sim_debug_kw_finish(buf) <= 0:
        print("not a KW_TAIL build"); sys.exit(0)
    f = np.array(buf[:2368], dtype=np.float64)
    f = f[f > 0]
    f = (f - f.min()) / 1e3
    spreads.append(f)
f = spreads[-1]
print(f"CTA finish spread (us after the first): p10 {np.percentile(f,10):.1f} p50 {np.percentile(f,50):.1f} "
      f"p90 {np.percentile(f,90):.1f} max {f.max():.1f}; mean idle before the end {f.max() - f.mean():.1f}")
