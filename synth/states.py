"""Seeded random valid simulation states for one-step parity tests.

A state is a dict in the layout shared by `sim_load_state` and the oracle's
`or_load_state`: vid-indexed status / lane / cursor / wait_steps / insert_time
/ arrive_time / s / v, junction-indexed policy / phase / elapsed / yellow_left /
pending, lane-indexed lane_dir, and the clock t.  Values are fp32-representable.
No model arithmetic here: only placement consistent with the trips' routes.
"""
from __future__ import annotations

import numpy as np

from .networks import KIND_DYNAMIC, KIND_TIDAL, POLICY_FIXED, POLICY_MANUAL, POLICY_MAXP, POLICY_NONE


def random_state(scen, seed=0, t=None, frac_driving=0.6, frac_pending=0.25,
                 tie_frac=0.15, overlap_frac=0.05, max_speed_factor=1.1,
                 junction_frac=0.25):
    rng = np.random.default_rng(seed)
    g, tr = scen.graph, scen.trips
    n = scen.n_trips
    nl = scen.n_lanes
    L = g["lane_length"]
    vmax = g["lane_max_speed"]
    lane_road = g["lane_road"]
    succ_off, succ = g["succ_offsets"], g["succ_lanes"]
    road_off, road_lanes = g["road_lane_offsets"], g["road_lanes"]
    roff, rroads = tr["route_offsets"], tr["route_roads"]
    nj = g["junc_lane_offsets"].shape[0] - 1
    if t is None:
        t = int(rng.integers(0, 500))
    status = np.full(n, 2, np.uint8)
    u = rng.random(n)
    status[u < frac_driving] = 1
    status[(u >= frac_driving) & (u < frac_driving + frac_pending)] = 0
    lane = np.full(n, -1, np.int32)
    cursor = np.zeros(n, np.int32)
    for k in np.where(status == 1)[0]:
        r = rroads[roff[k]:roff[k + 1]]
        c = int(rng.integers(len(r)))
        if c + 1 < len(r) and rng.random() < junction_frac:
            opts = []
            for l in road_lanes[road_off[r[c]]:road_off[r[c] + 1]]:
                for j in succ[succ_off[l]:succ_off[l + 1]]:
                    if lane_road[j] < 0 and lane_road[succ[succ_off[j]]] == r[c + 1]:
                        opts.append(j)
            if opts:
                lane[k] = opts[int(rng.integers(len(opts)))]
                cursor[k] = c
                continue
        ls = road_lanes[road_off[r[c]]:road_off[r[c] + 1]]
        lane[k] = ls[int(rng.integers(len(ls)))]
        cursor[k] = c
    s = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    drv = np.where(status == 1)[0]
    plen = scen.profiles[tr["profile"].astype(np.int64), 5]
    by_lane = {}
    for k in drv:
        by_lane.setdefault(int(lane[k]), []).append(int(k))
    for l, ks in by_lane.items():
        ks = list(rng.permutation(ks))
        Ll = float(L[l])
        need = sum(float(plen[k]) + 2.0 for k in ks)
        if need < Ll:
            slack = Ll - need
            cuts = np.sort(rng.uniform(0, slack, len(ks)))
            pos = 0.0
            prev = 0.0
            for i, k in enumerate(ks):
                pos += cuts[i] - prev
                prev = cuts[i]
                front = pos + float(plen[k])
                s[k] = np.float32(min(front, Ll))
                pos = front + 2.0
        else:
            for k in ks:
                s[k] = np.float32(rng.uniform(0, Ll))
    for k in drv:
        l = int(lane[k])
        x = rng.random()
        if x < tie_frac:                 # coarse grid -> equal-s ties across/within lanes
            s[k] = np.float32(np.round(s[k] / 5.0) * 5.0)
        elif x < tie_frac + overlap_frac:
            s[k] = np.float32(rng.uniform(0, float(L[l])))
        elif x < tie_frac + overlap_frac + 0.02:
            s[k] = L[l]                   # exactly at the stop line
        s[k] = np.float32(min(max(float(s[k]), 0.0), float(L[l])))
        y = rng.random()
        if y < 0.15:
            v[k] = 0.0
        else:
            v[k] = np.float32(rng.uniform(0, float(vmax[l]) * max_speed_factor))
    wait = rng.integers(0, 50, n).astype(np.int32)
    insert_time = np.where(status >= 1, rng.integers(0, t + 1, n), -1).astype(np.int32)
    arrive_time = np.where(status == 2, np.maximum(insert_time, 0) + rng.integers(1, 100, n),
                           -1).astype(np.int32)
    cursor[status != 1] = 0
    wait[status == 0] = 0
    # junction states
    pol0 = g["junc_policy"]
    nph = np.diff(g["junc_phase_offsets"])
    steps = g["phase_green_steps"]
    Y = scen.params["yellow_steps"]
    jpol = pol0.copy()
    jph = np.zeros(nj, np.int32)
    jel = np.zeros(nj, np.int32)
    jy = np.zeros(nj, np.int32)
    jpe = np.zeros(nj, np.int32)
    jrem = np.full(nj, -1, np.int32)
    for j in range(nj):
        K = int(nph[j])
        if K == 0:
            jpol[j] = POLICY_NONE
            continue
        if pol0[j] != POLICY_NONE and rng.random() < 0.25:
            jpol[j] = POLICY_MANUAL
        p = int(rng.integers(K))
        jph[j] = p
        if jpol[j] == POLICY_FIXED:
            g_p = int(steps[g["junc_phase_offsets"][j] + p])
            jel[j] = int(rng.integers(g_p))
            if rng.random() < 0.3 and Y > 0:
                jy[j] = int(rng.integers(1, Y + 1))
                jel[j] = g_p
            jpe[j] = (p + 1) % K if jy[j] > 0 else p
        elif jpol[j] == POLICY_MAXP:
            per = int(scen.params.get("max_pressure_period", 30))
            jel[j] = per - 1 if rng.random() < 0.6 else int(rng.integers(per))
            if rng.random() < 0.2 and Y > 0:
                jy[j] = int(rng.integers(1, Y + 1))
                jel[j] = per
                jpe[j] = int(rng.integers(K))
            else:
                jpe[j] = p
        elif jpol[j] == POLICY_MANUAL:
            jel[j] = int(rng.integers(100))
            if rng.random() < 0.4:                     # a set_tl_duration timer running
                jrem[j] = int(rng.integers(1, 4))
            if rng.random() < 0.3 and Y > 0:
                jy[j] = int(rng.integers(1, Y + 1))
                jpe[j] = int(rng.integers(K))
            else:
                jpe[j] = p
    ldir = g["lane_dir0"].copy()
    kinds = g["lane_kind"]
    part = g["tidal_partner"]
    for l in range(nl):
        if kinds[l] == KIND_DYNAMIC:
            ldir[l] = rng.integers(2)
        elif kinds[l] == KIND_TIDAL and part[l] > l:
            d = int(rng.integers(2))
            ldir[l], ldir[part[l]] = d, 1 - d
    return dict(t=int(t), status=status, lane=lane, cursor=cursor, wait_steps=wait,
                insert_time=insert_time, arrive_time=arrive_time, s=s, v=v,
                junc_policy=jpol.astype(np.uint8), junc_phase=jph, junc_elapsed=jel,
                junc_yellow_left=jy, junc_pending=jpe, junc_remaining=jrem,
                lane_dir=ldir.astype(np.uint8),
                lane_signal=np.zeros(nl, np.uint8))
