"""Diagnostic for the intermittent loopback lane_offsets mismatch:
partitioned runs of the city scenario of test_partition_invariance, checking
the lane order of sim_read_state for duplicates / missing vehicles against the
per-vehicle lanes (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
import paper_2406_10661_b200 as p
scen = synth.city(G=12, n_vehicles=20000, seed=13)
ref = p.Sim.from_scenario(scen)
ref.step(150)
r = ref.read_state(lane_order=True)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    for world, direct in ((3, False), (5, False), (5, True)):
        g = p.Sim.from_scenario(scen, world=world, loopback=True, direct=direct)
        g.step(150)
        s = g.read_state(lane_order=True)
        if np.array_equal(s["lane_offsets"], r["lane_offsets"]):
            g.destroy(); continue
        order = s["lane_order"][:s["lane_offsets"][-1]]
        u, c = np.unique(order, return_counts=True)
        dup = u[c > 1]
        drv = np.nonzero(s["status"] == 1)[0]
        missing = np.setdiff1d(drv, order)
        lanes_of = np.repeat(np.arange(len(s["lane_offsets"]) - 1), np.diff(s["lane_offsets"]))
        print(f"it {it} world {world} direct {direct}: listed {len(order)} driving {len(drv)} "
              f"dups {dup[:10]} missing {missing[:10]}", flush=True)
        for v in dup[:3]:
            where = lanes_of[np.nonzero(order == v)[0]]
            print(f"   vid {v}: listed in lanes {where}, state lane {s['lane'][v]}, ref lane {r['lane'][v]}, s {s['s'][v]}")
        per_ref = np.diff(r["lane_offsets"]); per = np.diff(s["lane_offsets"])
        bad = np.nonzero(per != per_ref)[0]
        print("   lanes with different counts:", bad[:10], per[bad[:10]], per_ref[bad[:10]])
        g.destroy()
print("done", flush=True)
