"""Pins of the CPU oracle against what the paper and mathematics fix.

Every expected value comes from tests/golden/oracle_pins.json (paper formulas,
closed forms, published known-answer vectors, hand-checked worked examples,
each with its citation) or from a closed form solved here independently of
oracle/.  None comes from the oracle or the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import synth
from synth import NetBuilder, Scenario, default_profiles, default_params

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_pins.json")))
V0 = float(np.float32(16.667))


def test_idm_closed_forms(oracle_lib):
    o = oracle_lib
    assert o.idm(0.0, V0, False, 0.0, 0.0) == GOLD["P-IDM-1"]["expect_a"]
    assert o.idm(V0, V0, False, 0.0, 0.0) == GOLD["P-IDM-2"]["expect_a"]
    p3 = GOLD["P-IDM-3"]
    assert abs(o.idm(p3["v"], V0, True, p3["gap"], p3["dv"]) - p3["expect_a"]) < p3["tol"]
    p4 = GOLD["P-SIG-1"]
    assert abs(o.idm(p4["v"], V0, True, p4["gap"], p4["dv"]) - p4["expect_a"]) < p4["tol"]


def test_idm_special_cases(oracle_lib):
    o = oracle_lib
    # ledger L8: zero / negative gap -> -b_hard without division
    assert o.idm(5.0, V0, True, 0.0, 0.0) == -8.0
    assert o.idm(5.0, V0, True, -3.0, 0.0) == -8.0
    # clamp at -b_hard for a tiny gap
    assert o.idm(15.0, V0, True, 0.01, 15.0) == -8.0
    # monotone: increasing in gap, decreasing in dv
    gaps = np.linspace(0.5, 200, 50)
    a = [o.idm(10.0, V0, True, g, 0.0) for g in gaps]
    assert all(x <= y for x, y in zip(a, a[1:]))
    dvs = np.linspace(-5, 5, 41)
    a = [o.idm(10.0, V0, True, 30.0, d) for d in dvs]
    assert all(x >= y for x, y in zip(a, a[1:]))
    # never above a_max
    for v in (0.0, 3.0, 10.0, 16.0):
        for g in (0.5, 5.0, 50.0, 500.0):
            assert o.idm(v, V0, True, g, -3.0) <= 2.0


def test_p_lc(oracle_lib):
    o = oracle_lib
    m = GOLD["P-MOB-1"]
    assert abs(o.p_lc(m["u_total"]) - m["expect_p"]) < m["tol"]
    for u, p in GOLD["P-MOB-2"]["cases"]:
        assert o.p_lc(u) == p
    # literal piecewise (L14): one-sided limit at 0+ is 0 while p_LC(0) = 2e-8
    # (S:278); at 1- it is 0.9 - 2e-8 while p_LC(1) = 0.9
    assert o.p_lc(1e-12) < 1e-11
    assert abs(o.p_lc(1.0 - 1e-12) - (0.9 - 2e-8)) < 1e-12


def test_philox_kat(oracle_lib):
    def h(x):
        return int(x, 16) if isinstance(x, str) else int(x)
    for c in GOLD["P-RNG"]["cases"]:
        out = oracle_lib.philox4x32_10([h(x) for x in c["ctr"]], [h(x) for x in c["key"]])
        assert [int(x) for x in out] == [h(x) for x in c["out"]]


def test_u53_range_and_uniformity(oracle_lib):
    r = np.array([oracle_lib.u53(7, k, t) for k in range(200) for t in range(20)])
    assert r.min() >= 0.0 and r.max() < 1.0
    assert abs(r.mean() - 0.5) < 0.02
    # 53-bit resolution: values are integer multiples of 2^-53
    assert all(float(x * 2.0 ** 53).is_integer() for x in r[:100])


def _equilibrium_speed(gap, v0=V0, s0=2.0, T=1.5):
    """Root of gap = (s0 + vT)/sqrt(1-(v/v0)^4) by bisection (closed form of
    the IDM equilibrium, P:158-161 with a = 0, dv = 0)."""
    lo, hi = 0.0, v0 * (1 - 1e-15)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        f = (s0 + mid * T) / np.sqrt(1 - (mid / v0) ** 4) - gap
        if f > 0:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def test_equilibrium_ring_c1(oracle_lib):
    eq = GOLD["P-EQ"]
    s = synth.ring(n_vehicles=20, length=eq["ring_length"])
    o = oracle_lib.Oracle(s)
    o.step(eq["steps"])
    st = o.read_state()
    ve = dict(eq["sweep"])[20]
    assert abs(_equilibrium_speed(45.0) - ve) < 1e-7
    assert np.all(np.abs(st["v"] - ve) < 1e-6)
    # all gaps 45 m (ring: consecutive positions modulo L)
    ss = np.sort(st["s"])
    gaps = np.diff(np.concatenate([ss, [ss[0] + 1000.0]])) - 5.0
    assert np.all(np.abs(gaps - 45.0) < 1e-6)


@pytest.mark.parametrize("n,ve", [tuple(x) for x in GOLD["P-EQ"]["sweep"]])
def test_equilibrium_sweep(oracle_lib, n, ve):
    gap = 1000.0 / n - 5.0
    assert abs(_equilibrium_speed(gap) - ve) < 2e-7
    s = synth.ring(n_vehicles=n, length=1000.0)
    o = oracle_lib.Oracle(s)
    o.step(2000)
    st = o.read_state()
    assert np.all(np.abs(st["v"] - ve) < 1e-5 * max(1.0, ve))


def _single_road(L, s_start, v_start, lanes=1, on_net=True, depart=0):
    b = NetBuilder()
    b.add_road(lanes, L, 16.667)
    trips = dict(depart_step=np.array([depart], np.int32),
                 on_network_at_t0=np.array([int(on_net)], np.uint8),
                 route_offsets=np.array([0, 1], np.int32), route_roads=np.zeros(1, np.int32),
                 start_lane=np.zeros(1, np.int32), start_s=np.array([s_start], np.float32),
                 start_v=np.array([v_start], np.float32), end_s=np.array([L], np.float32),
                 profile=np.zeros(1, np.uint8))
    return Scenario("road", b.graph(), trips, default_profiles(), default_params(1))


def _travel(o, horizon=500):
    for _ in range(horizon):
        o.step(1)
        m = o.metrics()
        if m["n_finished"]:
            return m["sum_travel_steps"]
    return None


def test_free_flow_travel_time(oracle_lib):
    ff = GOLD["P-FF"]
    for L, steps in ff["at_speed"]:
        tt = _travel(oracle_lib.Oracle(_single_road(L, 0.0, V0)))
        assert tt == steps and tt >= L / V0
    for L, steps in ff["from_rest"]:
        tt = _travel(oracle_lib.Oracle(_single_road(L, 0.0, 0.0)))
        assert tt == steps and tt >= L / V0


def test_one_step_from_rest(oracle_lib):
    o = oracle_lib.Oracle(_single_road(300.0, 10.0, 0.0))
    o.step(1)
    st = o.read_state()
    assert st["v"][0] == GOLD["P-STEP"]["v1"]
    assert st["s"][0] == 10.0 + GOLD["P-STEP"]["s1"]


def test_gold_two_lane_composition(oracle_lib):
    g = GOLD["P-GOLD-1"]
    b = NetBuilder()
    r = b.add_road(g["lanes"], g["road_length"], 16.667)
    veh = g["vehicles"]
    n = len(veh)
    trips = dict(depart_step=np.zeros(n, np.int32), on_network_at_t0=np.ones(n, np.uint8),
                 route_offsets=np.arange(n + 1).astype(np.int32),
                 route_roads=np.zeros(n, np.int32),
                 start_lane=np.array([b.road_lanes[r][x[0]] for x in veh], np.int32),
                 start_s=np.array([x[1] for x in veh], np.float32),
                 start_v=np.array([x[2] for x in veh], np.float32),
                 end_s=np.full(n, g["road_length"], np.float32), profile=np.zeros(n, np.uint8))
    sc = Scenario("gold", b.graph(), trips, default_profiles(), default_params(g["seed"]))
    for k, r_exp in enumerate(g["draws"]):
        assert abs(oracle_lib.u53(g["seed"], k, 0) - r_exp) < 1e-10
    o = oracle_lib.Oracle(sc)
    o.step(1)
    d = o.decisions()
    st = o.read_state()
    for k, (lc, lane_idx, s1, v1) in enumerate(g["expect"]):
        assert d["lc"][k] == lc
        assert st["lane"][k] == b.road_lanes[r][lane_idx]
        assert abs(st["s"][k] - s1) < g["tol"]
        assert abs(st["v"][k] - v1) < g["tol"]


def test_side_pointer_examples(oracle_lib):
    """L:{5,15}, R:{10}: for R@10 left_back = L@5, left_front = L@15;
    S:205: lane {v1@10, v2@20}: front(v1) = v2.  Equal s counts as back (L11)."""
    b = NetBuilder()
    b.add_road(2, 100.0, 16.667)
    pos = [(0, 15.0), (0, 25.0), (1, 20.0), (1, 30.0), (0, 30.0)]
    n = len(pos)
    trips = dict(depart_step=np.zeros(n, np.int32), on_network_at_t0=np.ones(n, np.uint8),
                 route_offsets=np.arange(n + 1).astype(np.int32), route_roads=np.zeros(n, np.int32),
                 start_lane=np.array([p[0] for p in pos], np.int32),
                 start_s=np.array([p[1] for p in pos], np.float32),
                 start_v=np.zeros(n, np.float32), end_s=np.full(n, 100.0, np.float32),
                 profile=np.zeros(n, np.uint8))
    o = oracle_lib.Oracle(Scenario("side", b.graph(), trips, default_profiles(), default_params(3)))
    o.step(1)
    d = o.decisions()
    sv = d["side_vid"]          # LF LB RF RB
    assert sv[2][0] == 1 and sv[2][1] == 0      # R@20: left front = L@25, left back = L@15
    assert d["leader_vid"][2] == 3              # front(v@20) = v@30 in the same lane
    assert sv[3][1] == 4 and sv[3][0] == -1     # R@30: L@30 has equal s -> back (L11)
    assert sv[4][3] == 3 and sv[4][2] == -1     # L@30: R@30 equal s -> right back
