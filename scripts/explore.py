"""Exploration: full-run aggregate agreement on C2 seeds + first C4 timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth, oracle
import paper_2406_10661_b200 as p
p.build()
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "c2"):
    for seed in (2, 3, 4, 5):
        sc = synth.grid(seed=seed)
        g = p.Sim.from_scenario(sc)
        o = oracle.Oracle(sc)
        g.step(3600); o.step(3600)
        mg, mo = g.read_metrics(), o.metrics()
        rel = lambda k: (mg[k] - mo[k]) / max(abs(mo[k]), 1e-9)
        print(f"C2 seed {seed}: fin {mg['n_finished']} vs {mo['n_finished']} ({rel('n_finished'):+.4f}) "
              f"att {mg['att_finished']:.2f} vs {mo['att_finished']:.2f} ({rel('att_finished'):+.4f}) "
              f"vs {rel('vehicle_steps'):+.4f} guard {mg['n_guard_hits']} / {mg['vehicle_steps']}", flush=True)
if what in ("all", "c4"):
    import torch
    t0 = time.time()
    sc = synth.city()
    print("gen", time.time() - t0, flush=True)
    t0 = time.time()
    g = p.Sim.from_scenario(sc)
    print("create", time.time() - t0, g.query_sizes(), flush=True)
    g.step(5); g.sync()
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.time()
        g.step(20); g.sync()
        dt = (time.time() - t0) / 20
        m = g.read_metrics()
        print(f"C4 step wall {dt*1e3:.3f} ms  -> {m['n_driving']/dt:.3e} veh-steps/s  guard {m['n_guard_hits']} of {m['vehicle_steps']} lc {m['n_lane_changes']} hand {m['n_handoffs']}", flush=True)
