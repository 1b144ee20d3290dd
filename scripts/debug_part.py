import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth
import paper_2406_10661_b200 as p
scen = synth.grid(rows=4, cols=4, road_len=250.0, lanes=2, n_trips=3000, seed=12, depart_window=400)
a = p.Sim.from_scenario(scen, record_decisions=True)
b = p.Sim.from_scenario(scen, record_decisions=True, world=2, loopback=True)
own, mig, halo = p.partition(scen.graph, scen.trips, scen.profiles, scen.params, 2)
lane_road = scen.graph["lane_road"]
def tile_of(l):
    if l < 0: return -1
    r = lane_road[l]
    if r >= 0: return r
    # junction lane: its predecessor's road
    so, sl = scen.graph["succ_offsets"], scen.graph["succ_lanes"]
    pred = np.where(sl == l)[0]
    src = np.searchsorted(so, pred[0], side='right') - 1
    return lane_road[src]
for t in range(150):
    sa0, sb0 = a.read_state(), b.read_state()
    a.step(1); b.step(1)
    sa, sb = a.read_state(), b.read_state()
    bad = [k for k in ("status","lane","s","v","cursor","wait_steps","insert_time","arrive_time") if not np.array_equal(sa[k], sb[k])]
    if bad:
        print("first diff at step", t, bad)
        for k in bad:
            idx = np.where(sa[k] != sb[k])[0][:5]
            for i in idx:
                print(k, "vid", i, "single:", sa["status"][i], sa["lane"][i], sa["s"][i], sa[k][i], " part:", sb["status"][i], sb["lane"][i], sb["s"][i], sb[k][i],
                      " prev lane", sa0["lane"][i], "prev s", sa0["s"][i], "prev status", sa0["status"][i],
                      " owner prev tile", own[tile_of(sa0["lane"][i])] if sa0["lane"][i]>=0 else None,
                      " owner new tile", own[tile_of(sa["lane"][i])] if sa["lane"][i]>=0 else None)
        da, db = a.read_decisions(), b.read_decisions()
        for i in idx:
            print("dec single", {k: da[k][i] for k in ("leader_vid","leader_hops","lc","handoffs","finished","inserted")})
            print("dec part  ", {k: db[k][i] for k in ("leader_vid","leader_hops","lc","handoffs","finished","inserted")})
        break
print("done")
