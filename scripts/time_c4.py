"""Quick device timing of k_step on C4 for a given library build (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2406_10661_b200.sim as S
lib = sys.argv[1] if len(sys.argv) > 1 else S.LIB
# SCALE=4: the 8M-vehicle instance of bench.py --scale 4 (G = 144)
scale = float(os.environ.get("SCALE", "1"))
cache = "/tmp/c4.npz" if scale == 1 else f"/tmp/c4_x{scale:g}.npz"
if os.path.exists(cache):
    scen = synth.load_scenario(cache)
else:
    scen = synth.city(G=int(round(72 * np.sqrt(scale))), n_vehicles=int(round(2_000_000 * scale)))
    synth.save_scenario(scen, cache)
S.load_library(lib)
st = torch.cuda.Stream()
sim = S.Sim.from_scenario(scen, stream=st.cuda_stream)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sim.step(int(os.environ.get("PREROLL", "10"))); sim.sync()
sim.enable_timing(True)
n = 40
m0 = sim.read_metrics()
with torch.cuda.stream(st):
    for k in range(n):
        flush.fill_(k & 255)
        sim.step(1)
torch.cuda.synchronize()
ks, sg, nl = sim.read_timing()
m1 = sim.read_metrics()
vs = m1["vehicle_steps"] - m0["vehicle_steps"]
print(f"{os.path.basename(lib)}: k_step {ks/n*1e3:.1f} us  k_signal {sg/n*1e3:.1f} us  "
      f"veh-steps/s(kstep) {vs/(ks/1e3):.3e}  guard/step {(m1['n_guard_hits']-m0['n_guard_hits'])/n:.0f}  "
      f"lc/step {(m1['n_lane_changes']-m0['n_lane_changes'])/n:.0f}  handoffs/step {(m1['n_handoffs']-m0['n_handoffs'])/n:.0f}  "
      f"driving {m1['n_driving']}", flush=True)
# sim_step(36): step graphs (6 steps per replay) with PDL, no flush between steps
sim.enable_timing(False)
with torch.cuda.stream(st):
    sim.step(36)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    sim.step(72)
    e1.record(st)
torch.cuda.synchronize()
print(f"  sim_step(72) (graphs): {e0.elapsed_time(e1) / 72 * 1e3:.1f} us per step", flush=True)
import ctypes
L = S.load_library(lib)
pb = (ctypes.c_ulonglong * 32)()
try:
    if L.sim_debug_kstep_prof(pb) > 0:
        # counters since the library was loaded: take a fresh window
        L.sim_debug_kstep_prof(pb)
        with torch.cuda.stream(st):
            for k in range(10):
                flush.fill_(k & 255)
                sim.step(1)
        torch.cuda.synchronize()
        L.sim_debug_kstep_prof(pb)
        names = {0: "P wait_empty", 1: "P build", 2: "P issue", 3: "P gather",
                 8: "C wait_full", 9: "C claim", 10: "C tile", 11: "C round barrier"}
        tot_p = sum(pb[i] for i in range(0, 5)); tot_c = sum(pb[i] for i in range(8, 19))
        for i, nm in names.items():
            tot = tot_p if i < 8 else tot_c
            print(f"  {nm:18s} {pb[i]/max(tot,1)*100:5.1f}%  ({pb[i]/1e6:.1f} Mcyc)")
        print(f"  tiles {pb[20]/10:.0f}/step  gmode {pb[21]/10:.0f}")
        ph = {22: "setup", 23: "merge", 24: "segs", 25: "pass1", 26: "pass2", 27: "pass3", 28: "fp64",
              29: "compact", 30: "finish"}
        tot = sum(pb[i] for i in ph) or 1
        print("  in tile: " + "  ".join(f"{nm} {pb[i]/tot*100:.1f}%" for i, nm in ph.items()))
        if pb[14]:
            print(f"  rounds {pb[14]}: slowest tile / mean tile = {pb[12]/max(pb[13],1):.2f}; vehicles of the slowest {pb[15]/pb[14]:.0f} vs mean {pb[16]/pb[14]:.0f}")
        tc = np.zeros(65536 * 4, np.uint32)
        if L.sim_debug_tile_cycles(tc.ctypes.data_as(ctypes.c_void_p)) > 0:
            tc = tc.reshape(-1, 4)[:scen.graph["road_lane_offsets"].shape[0] - 1]
            if os.environ.get("DUMP"):
                np.savez(os.environ["DUMP"], tc=tc)
                # a later step's per-tile cycles too (is the per-tile cost persistent?)
                sim.step(int(os.environ.get("DUMP_GAP", "1")))
                tc2 = np.zeros(65536 * 4, np.uint32)
                L.sim_debug_tile_cycles(tc2.ctypes.data_as(ctypes.c_void_p))
                np.savez(os.environ["DUMP"].replace(".npz", "_next.npz"),
                         tc=tc2.reshape(-1, 4)[:scen.graph["road_lane_offsets"].shape[0] - 1])
            cyc, nv = tc[:, 0].astype(float), tc[:, 1].astype(float)
            ok = (nv > 0) & (cyc > 0)
            if not ok.any():
                raise AttributeError("no per-tile cycles in this build")
            print(f"  tile cycles: mean {cyc[ok].mean():.0f} median {np.median(cyc[ok]):.0f} p90 {np.percentile(cyc[ok], 90):.0f} p99 {np.percentile(cyc[ok], 99):.0f}")
            per = cyc[ok] / nv[ok]
            print(f"  cycles/vehicle: mean {per.mean():.0f} median {np.median(per):.0f} p90 {np.percentile(per, 90):.0f} p99 {np.percentile(per, 99):.0f}")
            lc, hd = (tc[:, 2] & 0xffff)[ok], (tc[:, 2] >> 16)[ok]
            A_ = np.vstack([nv[ok], lc, hd, tc[ok, 3], np.ones(ok.sum())]).T
            coef = np.linalg.lstsq(A_, cyc[ok], rcond=None)[0]
            pred = A_ @ coef
            print("  fit cycles = %.0f*veh + %.0f*lc + %.0f*handoff + %.0f*lanes + %.0f ; R2 %.2f" % (*coef, 1 - ((cyc[ok]-pred)**2).sum()/((cyc[ok]-cyc[ok].mean())**2).sum()))
except AttributeError:
    pass
buf = (ctypes.c_ulonglong * 32)()
try:
    n = L.sim_debug_guard_stats(buf)
    if n > 0:
        names = ["idm_gap", "lim_select", "l19", "b_safe", "lane_start", "front_gap", "r_vs_p",
                 "uL_vs_uR", "clamp_bind", "clamp_overlap", "arrival", "handoff", "wait"]
        print({names[i]: buf[i] for i in range(len(names))})
        print("want", buf[20], "admissible", buf[21], "evaluated", buf[22], "vehicles", buf[23])
except AttributeError:
    pass
