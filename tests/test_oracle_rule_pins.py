"""Rule pins of the CPU oracle (VERDICT r01 "What's missing" #2): departure
insertion, the lane group and mandatory change (L18/L37),
the junction-lane choice (L24), the lookahead gap through a junction lane
(P:168-169, L9), the in-step stop of the integrator (L1) and several lanes in
one step (L31).

Expected values: tests/golden/rule_pins.json (hand-derived, each with its
citation and arithmetic) or closed forms evaluated here from the paper's IDM
(itself pinned by test_oracle_pins.py).  The scenarios are tiny
hand-built graphs (tests/pin_scenarios.py).  scripts/oracle_mutations.py
breaks the oracle once per rule and shows that one of these tests fails.
"""
import json
import math
import os

import numpy as np
import pytest

import pin_scenarios as PS

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rule_pins.json")))
V0 = float(np.float32(16.667))
PENDING, DRIVING, FINISHED = 0, 1, 2


def idm_closed(v, gap, dv, a_max=2.0, a_comf=3.0, T=1.5, s0=2.0, v0=V0, b_hard=8.0, lead=True):
    """P:158-161 (delta = 4), ledger L7/L8: the equation as printed."""
    free = 1.0 - (v / v0) ** 4
    if not lead:
        return max(a_max * free, -b_hard)
    ss = s0 + max(0.0, v * T + v * dv / (2.0 * math.sqrt(a_max * a_comf)))
    return max(a_max * (free - (ss / gap) ** 2), -b_hard)


def run(oracle_lib, scen, steps, K=None):
    o = oracle_lib.Oracle(scen, lookahead=K)
    o.step(steps)
    return o


# ---- O10 departures (L25) ----------------------------------------------
def _ins(oracle_lib, key, steps):
    g = GOLD[key]
    scen, _ = PS.insertion(g.get("obstacles", []), g["pending"])
    return run(oracle_lib, scen, steps), len(g.get("obstacles", []))


@pytest.mark.parametrize("key", ["INS-ACCEPT", "INS-AHEAD-REFUSE", "INS-AHEAD-BOUNDARY"])
def test_insertion_ahead_rule(oracle_lib, key):
    g = GOLD[key]
    o, _ = _ins(oracle_lib, key, g["steps"])
    st = o.read_state()
    for vid, t_ins in g["expect_insert_time"].items():
        vid = int(vid)
        assert st["status"][vid] == DRIVING and st["insert_time"][vid] == t_ins, (key, st["insert_time"])
    if "expect_s" in g:
        assert st["s"][1] == g["expect_s"] and st["v"][1] == 0.0
    # one step earlier the refused vehicle is still pending
    if g["expect_insert_time"]["1"] > 1:
        o2, _ = _ins(oracle_lib, key, g["expect_insert_time"]["1"] - 1)
        assert o2.read_state()["status"][1] == PENDING


@pytest.mark.parametrize("key", ["INS-BEHIND-ACCEPT", "INS-BEHIND-REFUSE"])
def test_insertion_behind_rule(oracle_lib, key):
    g = GOLD[key]
    o, nobs = _ins(oracle_lib, key, 1)
    st = o.read_state()
    assert (st["status"][nobs] == DRIVING) == g["expect_inserted_step0"], key
    assert bool(o.decisions()["inserted"][nobs]) == g["expect_inserted_step0"]


def test_insertion_lane_start_margin(oracle_lib):
    g = GOLD["INS-MARGIN"]
    ok, _ = PS.insertion([], [(0, g["accept_start_s"], 0)])
    no, _ = PS.insertion([], [(0, g["refuse_start_s"], 0)])
    assert run(oracle_lib, ok, 1).read_state()["status"][0] == DRIVING
    assert run(oracle_lib, no, 5).read_state()["status"][0] == PENDING


def test_insertion_priority_depart_then_vid(oracle_lib):
    g = GOLD["INS-PRIORITY"]
    scen, _ = PS.insertion([], g["pending"])
    o = run(oracle_lib, scen, 6)
    st = o.read_state()
    assert st["status"][1] == DRIVING and st["insert_time"][1] == g["expect_insert_time_vid1"]
    assert st["status"][0] == PENDING or st["insert_time"][0] > g["expect_insert_time_vid1"]
    # ties in depart: lower vid first
    scen, _ = PS.insertion([], GOLD["INS-TIE"]["pending"])
    st = run(oracle_lib, scen, 1).read_state()
    assert st["status"][0] == DRIVING and st["status"][1] == PENDING


def test_insertion_one_per_lane(oracle_lib):
    g = GOLD["INS-ONE-PER-LANE"]
    scen, _ = PS.insertion([], g["pending"])
    st = run(oracle_lib, scen, 2).read_state()
    assert list(st["insert_time"]) == g["expect_insert_time"]
    g = GOLD["INS-TWO-LANES"]
    scen, _ = PS.insertion([], g["pending"], lanes=2)
    st = run(oracle_lib, scen, 1).read_state()
    assert list(st["insert_time"]) == g["expect_insert_time"]


# ---- lane group and mandatory change (L18, L37) ---------------------------
@pytest.mark.parametrize("key", ["MAND-LEFT", "MAND-RIGHT", "MAND-L37-TIE"])
def test_mandatory_change(oracle_lib, key):
    g = GOLD[key]
    seed = PS.seed_with_draw_above(g["draw_above"])
    li, s, v = g["ego"]
    scen, lanes = PS.mandatory(g["n_lanes"], g["group"], li, s, v, seed)
    o = run(oracle_lib, scen, 1)
    assert o.decisions()["lc"][0] == g["expect_lc"]
    assert o.read_state()["lane"][0] == lanes[g["expect_lane_idx"]]


def test_mandatory_stop_line(oracle_lib):
    g = GOLD["MAND-STOPLINE"]
    li, s, v = g["ego"]
    scen, lanes = PS.mandatory(g["n_lanes"], g["group"], li, s, v, seed=1,
                               others=[tuple(x) for x in g["others"]], red=True, L=g["L"])
    o = oracle_lib.Oracle(scen)
    for _ in range(g["steps"]):
        o.step(1)
        st = o.read_state()
        assert st["status"][0] == DRIVING and st["lane"][0] == lanes[li]
        assert st["s"][0] <= g["L"]
        assert o.decisions()["phantom"][0] == 1
    # it advanced to the stop line: IDM against the stationary phantom at L
    # settles at the jam gap s0 = 2 (P:158-161 with v = 0)
    # (the ballistic update overshoots it by a few cm on the way in)
    assert abs(st["s"][0] - (g["L"] - 2.0)) < 0.1


# ---- junction-lane choice (L24) ------------------------------------------------------
@pytest.mark.parametrize("dest", ["D", "C", "B", "X"])
def test_exit_lane_choice(oracle_lib, dest):
    scen, js = PS.exit_choice(dest)
    st = run(oracle_lib, scen, 1).read_state()
    assert st["lane"][0] == js[GOLD["EXIT-CHOICE"]["expect"][dest]], dest


# ---- lookahead gap through a junction lane (L9) -----------------------------
@pytest.mark.parametrize("K", [1, 2])
def test_lookahead_through_junction_lane(oracle_lib, K):
    g = GOLD["LOOK-H2"]
    scen, _ = PS.lookahead(K, g["L_a"], g["L_j"], tuple(g["ego"]), tuple(g["lead"]))
    o = run(oracle_lib, scen, 1, K=K)
    d = o.decisions()
    v, vf = g["ego"][1], g["lead"][1]
    if K == 2:
        assert d["leader_vid"][0] == 1 and d["leader_hops"][0] == g["expect_hops_K2"]
        a = idm_closed(v, g["expect_gap"], v - vf)
    else:
        assert d["leader_vid"][0] == -1 and d["leader_hops"][0] == g["expect_hops_K1"]
        a = idm_closed(v, 0.0, 0.0, lead=False)
    assert abs(d["accel"][0] - a) <= 1e-12 * max(1.0, abs(a))
    st = o.read_state()
    assert abs(st["s"][0] - (g["ego"][0] + (v + (v + a)) / 2.0)) <= 1e-12 * 100


# ---- integrator: in-step stop (L1) -----------------------------------------------------
def test_stop_within_step(oracle_lib):
    g = GOLD["STOP-IN-STEP"]
    (s, v), (sl, vl) = g["ego"], g["lead"]
    assert idm_closed(v, (sl - s) - 5.0, v - vl) == g["expect_a"]      # clamp binds
    o = run(oracle_lib, PS.stop_in_step(tuple(g["ego"]), tuple(g["lead"])), 1)
    assert o.decisions()["accel"][0] == g["expect_a"]
    st = o.read_state()
    assert st["s"][0] == g["expect_s"] and st["v"][0] == g["expect_v"]


# ---- several lanes in one step (L31) ---------------------------------------------------
def test_two_lane_crossing_in_one_step(oracle_lib):
    g = GOLD["CROSS-TWO"]
    s, v = g["ego"]
    scen, (a0, j, b0) = PS.crossing(tuple(g["ego"]), g["L_j"])
    o = run(oracle_lib, scen, 1)
    st, d = o.read_state(), o.decisions()
    a = idm_closed(v, 0.0, 0.0, lead=False)
    s1 = ((s + (v + (v + a)) / 2.0) - 100.0) - g["L_j"]
    assert d["handoffs"][0] == g["expect_handoffs"]
    assert st["lane"][0] == b0 and st["cursor"][0] == g["expect_cursor"]
    assert abs(st["s"][0] - s1) <= 1e-12 * 100


# ---- ATT over all vehicles (ledger L27) ---------------------------------------
def test_att_all_counts_trips_in_progress(oracle_lib):
    """P:876 'the average time taken by all vehicles': a finished trip counts
    its travel time, a trip in progress its time so far.  Two unconnected
    roads: vid 0 drives 1000 m at v0 from t = 0 (travel 60 steps, P-FF of
    oracle_pins.json); vid 1 departs at t = 0 on a 5000 m road (inserted at
    t = 1).  At t = 70: ATT_all = (60 + (70 - 1)) / 2."""
    import json, os
    ff = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_pins.json")))["P-FF"]
    L1, travel = ff["at_speed"][0]
    b = PS.NetBuilder()
    A = b.add_road(1, L1, PS.VMAX)
    B = b.add_road(1, 5000.0, PS.VMAX)
    rows = [dict(route=[A], lane=b.road_lanes[A][0], s=0.0, v=V0, end_s=L1),
            dict(route=[B], lane=b.road_lanes[B][0], s=30.0, v=0.0, depart=0, on_net=0, end_s=5000.0)]
    o = run(oracle_lib, PS.scenario("att", b, rows), 70)
    m = o.metrics()
    assert m["n_finished"] == 1 and m["n_driving"] == 1
    assert m["att_finished"] == travel
    assert m["sum_time_driving"] == 70 - 1
    assert m["att_all"] == (travel + (70 - 1)) / 2
