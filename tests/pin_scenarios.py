"""Tiny hand-built scenarios for the rule pins of tests/test_oracle_rule_pins.py
(oracle, -m "not gpu") and tests/test_gpu_rule_pins.py (CUDA path, K = 1 and
K = 2).  Graph construction and trip arrays only: no model arithmetic here.

Every scenario uses the default profile (a_max 2, a_comf 3, T 1.5, s0 2,
v_max 16.667, length 5; ledger L4) unless stated, so
v0 = fp32(16.667) = 16.666999816894531 and the lane-start margin (L17) is
v_cap + 0.5 * a_cap = 16.666999816894531 + 1.0.
"""
from __future__ import annotations

import numpy as np

from synth import NetBuilder, Scenario, default_profiles, default_params  # noqa: F401 (re-exported)
from synth.networks import POLICY_FIXED, POLICY_NONE, TURN_LEFT, TURN_RIGHT, TURN_STRAIGHT

VMAX = 16.667


def trips(rows):
    """rows: dicts with route (road ids), lane, s, v, depart (default 0),
    on_net (default 1), end_s, profile (default 0)."""
    n = len(rows)
    routes = [list(r["route"]) for r in rows]
    off = np.zeros(n + 1, np.int32)
    off[1:] = np.cumsum([len(r) for r in routes])
    return dict(
        depart_step=np.array([r.get("depart", 0) for r in rows], np.int32),
        on_network_at_t0=np.array([r.get("on_net", 1) for r in rows], np.uint8),
        route_offsets=off,
        route_roads=np.array([x for r in routes for x in r], np.int32),
        start_lane=np.array([r["lane"] for r in rows], np.int32),
        start_s=np.array([r["s"] for r in rows], np.float32),
        start_v=np.array([r.get("v", 0.0) for r in rows], np.float32),
        end_s=np.array([r["end_s"] for r in rows], np.float32),
        profile=np.array([r.get("profile", 0) for r in rows], np.uint8))


def two_profiles():
    """default profile (row 0) + a slow long one (row 1: a_max 1, length 7)."""
    return np.concatenate([default_profiles(),
                           np.array([[1.0, 3.0, 1.5, 2.0, 16.667, 7.0]], np.float32)])


def scenario(name, b, rows, seed=1, lookahead=2, profiles=None):
    p = default_params(seed)
    p["lookahead_lanes"] = lookahead
    prof = default_profiles() if profiles is None else profiles
    return Scenario(name, b.graph(), trips(rows), prof, p)


# ---------------------------------------------------------------------------
# O10 departures (ledger L25)
# ---------------------------------------------------------------------------
def insertion(obstacles, pending, L=300.0, lanes=1):
    """One road; `obstacles` = [(lane_idx, s, v[, profile])] DRIVING at t = 0
    (vids first), `pending` = [(lane_idx, start_s, depart)] PENDING with the
    default profile; every trip ends at L.  Profiles: two_profiles()."""
    b = NetBuilder()
    r = b.add_road(lanes, L, VMAX)
    ln = b.road_lanes[r]
    rows = [dict(route=[r], lane=ln[o[0]], s=o[1], v=o[2], profile=(o[3] if len(o) > 3 else 0),
                 end_s=L) for o in obstacles]
    rows += [dict(route=[r], lane=ln[li], s=s, v=0.0, depart=d, on_net=0, end_s=L)
             for li, s, d in pending]
    return scenario("ins", b, rows, profiles=two_profiles()), ln


# ---------------------------------------------------------------------------
# lane group and mandatory change (ledger L18, L37)
# ---------------------------------------------------------------------------
def mandatory(n_lanes, group_lanes, ego_lane, ego_s, ego_v, seed, others=(), red=False,
              L=200.0):
    """Road A (n_lanes, length L) -> junction J -> road B (1 lane) from the
    lanes in `group_lanes`, and -> road C (1 lane) from every other lane of A.
    The ego (vid 0) has route [A, B]; `others` = [(lane_idx, s, v)] with
    route [A, B] too.  red: J runs FIXED_TIME with the movements into B red
    for 10,000 steps (phase 0 = the movements into C)."""
    b = NetBuilder()
    A = b.add_road(n_lanes, L, VMAX)
    B = b.add_road(1, 300.0, VMAX)
    Cr = b.add_road(1, 300.0, VMAX)
    J = b.add_junction(policy=POLICY_FIXED if red else POLICY_NONE)
    to_b, to_c = [], []
    for i, a in enumerate(b.road_lanes[A]):
        if i in group_lanes:
            to_b.append(b.connect(J, a, b.road_lanes[B][0], TURN_STRAIGHT, 20.0, VMAX))
        else:
            to_c.append(b.connect(J, a, b.road_lanes[Cr][0], TURN_RIGHT, 20.0, VMAX))
    if red:
        b.set_phases(J, [set(to_c), set(to_b)], [10000, 10])
    rows = [dict(route=[A, B], lane=b.road_lanes[A][ego_lane], s=ego_s, v=ego_v, end_s=300.0)]
    rows += [dict(route=[A, B], lane=b.road_lanes[A][li], s=s, v=v, end_s=300.0)
             for li, s, v in others]
    return scenario("mand", b, rows, seed=seed), b.road_lanes[A]


# ---------------------------------------------------------------------------
# junction-lane choice (ledger L24)
# ---------------------------------------------------------------------------
def exit_choice(dest):
    """Road A (1 lane, 100 m) -> J1 -> road B (3 lanes, 300 m): a0 -> b0 via
    junction lane j0, a0 -> b1 via j1 (j0 < j1); J2: b0 -> C, b1 -> D, b2 -> X.
    The ego starts at s = 95, v = 10 on a0 with route [A, B, dest] (dest in
    'B' (destination road), 'C', 'D', 'X') and enters the junction in step 0."""
    b = NetBuilder()
    A = b.add_road(1, 100.0, VMAX)
    B = b.add_road(3, 300.0, VMAX)
    roads = {nm: b.add_road(1, 300.0, VMAX) for nm in ("C", "D", "X")}
    J1 = b.add_junction(policy=POLICY_NONE)
    J2 = b.add_junction(policy=POLICY_NONE)
    a0 = b.road_lanes[A][0]
    bl = b.road_lanes[B]
    j0 = b.connect(J1, a0, bl[0], TURN_LEFT, 20.0, VMAX)
    j1 = b.connect(J1, a0, bl[1], TURN_STRAIGHT, 20.0, VMAX)
    b.connect(J2, bl[0], b.road_lanes[roads["C"]][0], TURN_LEFT, 20.0, VMAX)
    b.connect(J2, bl[1], b.road_lanes[roads["D"]][0], TURN_STRAIGHT, 20.0, VMAX)
    b.connect(J2, bl[2], b.road_lanes[roads["X"]][0], TURN_RIGHT, 20.0, VMAX)
    route = [A, B] if dest == "B" else [A, B, roads[dest]]
    rows = [dict(route=route, lane=a0, s=95.0, v=10.0, end_s=300.0)]
    return scenario("exit", b, rows), (j0, j1)


# ---------------------------------------------------------------------------
# lookahead through a junction lane (ledger L9)
# ---------------------------------------------------------------------------
def lookahead(K, L_a=100.0, L_j=20.0, ego=(60.0, 10.0), lead=(30.0, 10.0)):
    """Road A (1 lane, L_a) -> junction lane (L_j, empty, GREEN) -> road B
    (1 lane, 200 m).  Ego (vid 0) on A at ego = (s, v), route [A, B]; the only
    vehicle on B (vid 1) at lead = (s, v), route [B]."""
    b = NetBuilder()
    A = b.add_road(1, L_a, VMAX)
    B = b.add_road(1, 200.0, VMAX)
    J = b.add_junction(policy=POLICY_NONE)
    j = b.connect(J, b.road_lanes[A][0], b.road_lanes[B][0], TURN_STRAIGHT, L_j, VMAX)
    rows = [dict(route=[A, B], lane=b.road_lanes[A][0], s=ego[0], v=ego[1], end_s=200.0),
            dict(route=[B], lane=b.road_lanes[B][0], s=lead[0], v=lead[1], end_s=200.0)]
    return scenario("look", b, rows, lookahead=K), (b.road_lanes[A][0], j, b.road_lanes[B][0])


# ---------------------------------------------------------------------------
# integrator branches (ledger L1) and multi-lane crossing (L31)
# ---------------------------------------------------------------------------
def stop_in_step(ego=(100.0, 4.0), lead=(110.0, 0.0), K=2):
    """One road (300 m): ego (vid 0) closing on a stationary vehicle (vid 1)."""
    b = NetBuilder()
    r = b.add_road(1, 300.0, VMAX)
    ln = b.road_lanes[r][0]
    rows = [dict(route=[r], lane=ln, s=ego[0], v=ego[1], end_s=300.0),
            dict(route=[r], lane=ln, s=lead[0], v=lead[1], end_s=300.0)]
    return scenario("stop", b, rows, lookahead=K)


def crossing(ego=(95.0, 15.0), L_j=5.0, K=2):
    """Road A (100 m) -> junction lane of L_j m (GREEN) -> road B (200 m);
    the ego (vid 0, route [A, B]) crosses the whole junction lane in step 0."""
    b = NetBuilder()
    A = b.add_road(1, 100.0, VMAX)
    B = b.add_road(1, 200.0, VMAX)
    J = b.add_junction(policy=POLICY_NONE)
    j = b.connect(J, b.road_lanes[A][0], b.road_lanes[B][0], TURN_STRAIGHT, L_j, VMAX)
    rows = [dict(route=[A, B], lane=b.road_lanes[A][0], s=ego[0], v=ego[1], end_s=200.0)]
    return scenario("cross", b, rows, lookahead=K), (b.road_lanes[A][0], j, b.road_lanes[B][0])


# ---------------------------------------------------------------------------
# Philox4x32-10 written out here (independent of oracle/ and the CUDA path;
# pinned by the same published known-answer vectors, P-RNG) — used to pick
# seeds whose draw makes a discretionary change impossible
# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key):
    M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
    c = [x & 0xffffffff for x in ctr]
    k0, k1 = key[0] & 0xffffffff, key[1] & 0xffffffff
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        hi0, lo0 = p0 >> 32, p0 & 0xffffffff
        hi1, lo1 = p1 >> 32, p1 & 0xffffffff
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + W0) & 0xffffffff
        k1 = (k1 + W1) & 0xffffffff
    return c


def u53(seed, vid, t):
    """ledger L16: U53 of Philox4x32-10(key = seed; counter = (vid, t, 0, 0))."""
    x = philox4x32_10([vid, t, 0, 0], [seed & 0xffffffff, seed >> 32])
    return (((x[0] >> 5) << 26) + (x[1] >> 6)) * 2.0 ** -53


def seed_with_draw_above(threshold, vid=0, t=0):
    for seed in range(1, 10000):
        if u53(seed, vid, t) >= threshold:
            return seed
    raise RuntimeError("no seed")
