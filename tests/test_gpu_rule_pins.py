"""The rule pins of test_oracle_rule_pins.py run on the CUDA path (VERDICT r01
"Next round" #1: "a GPU run of the same cases in K = 1 paper-literal mode"):
departure insertion, the lane group and mandatory change
(L18/L37), the junction-lane choice (L24), the lookahead gap through
a junction lane (K = 1 paper-literal and K = 2), the in-step stop
(L1) and two lanes crossed in one step (L31).

Same tiny scenarios (tests/pin_scenarios.py), same hand-derived expectations
(tests/golden/rule_pins.json), through the C ABI, in both the fp32 + guard
default and exact_mode.  Integer outcomes must equal the expectation exactly;
positions / accelerations are the fp32 state of the expected fp64 value
(relative 1e-6)."""
import json
import math
import os

import numpy as np
import pytest

import pin_scenarios as PS

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rule_pins.json")))
V0 = float(np.float32(16.667))
PENDING, DRIVING = 0, 1
MODES = [False, True]                               # exact_mode


@pytest.fixture(scope="module")
def simlib():
    import paper_2406_10661_b200 as p
    p.build()
    return p


def idm_closed(v, gap, dv, a_max=2.0, a_comf=3.0, T=1.5, s0=2.0, v0=V0, b_hard=8.0, lead=True):
    """P:158-161 (delta = 4), ledger L7/L8, as printed."""
    free = 1.0 - (v / v0) ** 4
    if not lead:
        return max(a_max * free, -b_hard)
    ss = s0 + max(0.0, v * T + v * dv / (2.0 * math.sqrt(a_max * a_comf)))
    return max(a_max * (free - (ss / gap) ** 2), -b_hard)


def close(x, y, rel=1e-6):
    return abs(float(x) - float(y)) <= rel * max(1.0, abs(float(y)))


class Run:
    """One CUDA-path run of a pin scenario (decisions recorded)."""

    def __init__(self, simlib, scen, steps, exact):
        self.g = simlib.Sim.from_scenario(scen, exact_mode=exact, record_decisions=True)
        self.g.step(steps)

    def state(self):
        return self.g.read_state()

    def dec(self):
        return self.g.read_decisions()


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("key", ["INS-ACCEPT", "INS-AHEAD-REFUSE", "INS-AHEAD-BOUNDARY"])
def test_insertion_ahead_rule_gpu(simlib, key, exact):
    g = GOLD[key]
    scen, _ = PS.insertion(g.get("obstacles", []), g["pending"])
    st = Run(simlib, scen, g["steps"], exact).state()
    for vid, t_ins in g["expect_insert_time"].items():
        assert st["status"][int(vid)] == DRIVING and st["insert_time"][int(vid)] == t_ins, key
    if "expect_s" in g:
        assert st["s"][1] == g["expect_s"] and st["v"][1] == 0.0
    if g["expect_insert_time"]["1"] > 1:
        st2 = Run(simlib, scen, g["expect_insert_time"]["1"] - 1, exact).state()
        assert st2["status"][1] == PENDING


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("key", ["INS-BEHIND-ACCEPT", "INS-BEHIND-REFUSE"])
def test_insertion_behind_rule_gpu(simlib, key, exact):
    g = GOLD[key]
    scen, _ = PS.insertion(g["obstacles"], g["pending"])
    r = Run(simlib, scen, 1, exact)
    nobs = len(g["obstacles"])
    assert (r.state()["status"][nobs] == DRIVING) == g["expect_inserted_step0"], key
    assert bool(r.dec()["inserted"][nobs]) == g["expect_inserted_step0"]


@pytest.mark.parametrize("exact", MODES)
def test_insertion_margin_priority_one_per_lane_gpu(simlib, exact):
    g = GOLD["INS-MARGIN"]
    ok, _ = PS.insertion([], [(0, g["accept_start_s"], 0)])
    no, _ = PS.insertion([], [(0, g["refuse_start_s"], 0)])
    assert Run(simlib, ok, 1, exact).state()["status"][0] == DRIVING
    assert Run(simlib, no, 5, exact).state()["status"][0] == PENDING
    g = GOLD["INS-PRIORITY"]
    st = Run(simlib, PS.insertion([], g["pending"])[0], 6, exact).state()
    assert st["status"][1] == DRIVING and st["insert_time"][1] == g["expect_insert_time_vid1"]
    assert st["status"][0] == PENDING or st["insert_time"][0] > g["expect_insert_time_vid1"]
    st = Run(simlib, PS.insertion([], GOLD["INS-TIE"]["pending"])[0], 1, exact).state()
    assert st["status"][0] == DRIVING and st["status"][1] == PENDING
    g = GOLD["INS-ONE-PER-LANE"]
    st = Run(simlib, PS.insertion([], g["pending"])[0], 2, exact).state()
    assert list(st["insert_time"]) == g["expect_insert_time"]
    g = GOLD["INS-TWO-LANES"]
    st = Run(simlib, PS.insertion([], g["pending"], lanes=2)[0], 1, exact).state()
    assert list(st["insert_time"]) == g["expect_insert_time"]


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("key", ["MAND-LEFT", "MAND-RIGHT", "MAND-L37-TIE"])
def test_mandatory_change_gpu(simlib, key, exact):
    g = GOLD[key]
    seed = PS.seed_with_draw_above(g["draw_above"])
    li, s, v = g["ego"]
    scen, lanes = PS.mandatory(g["n_lanes"], g["group"], li, s, v, seed)
    r = Run(simlib, scen, 1, exact)
    assert r.dec()["lc"][0] == g["expect_lc"]
    assert r.state()["lane"][0] == lanes[g["expect_lane_idx"]]


@pytest.mark.parametrize("exact", MODES)
def test_mandatory_stop_line_gpu(simlib, exact):
    g = GOLD["MAND-STOPLINE"]
    li, s, v = g["ego"]
    scen, lanes = PS.mandatory(g["n_lanes"], g["group"], li, s, v, seed=1,
                               others=[tuple(x) for x in g["others"]], red=True, L=g["L"])
    sim = simlib.Sim.from_scenario(scen, exact_mode=exact, record_decisions=True)
    for _ in range(g["steps"]):
        sim.step(1)
        st = sim.read_state()
        assert st["status"][0] == DRIVING and st["lane"][0] == lanes[li]
        assert st["s"][0] <= g["L"]
        assert sim.read_decisions()["phantom"][0] == 1
    assert abs(st["s"][0] - (g["L"] - 2.0)) < 0.1


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("dest", ["D", "C", "B", "X"])
def test_exit_lane_choice_gpu(simlib, dest, exact):
    scen, js = PS.exit_choice(dest)
    st = Run(simlib, scen, 1, exact).state()
    assert st["lane"][0] == js[GOLD["EXIT-CHOICE"]["expect"][dest]], dest


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("K", [1, 2])
def test_lookahead_through_junction_lane_gpu(simlib, K, exact):
    """K = 1 is the paper-literal lookahead ('the first vehicle in the next
    lane'): the junction lane is empty, so there is no leader."""
    g = GOLD["LOOK-H2"]
    scen, _ = PS.lookahead(K, g["L_a"], g["L_j"], tuple(g["ego"]), tuple(g["lead"]))
    assert scen.params["lookahead_lanes"] == K
    r = Run(simlib, scen, 1, exact)
    d = r.dec()
    v, vf = g["ego"][1], g["lead"][1]
    if K == 2:
        assert d["leader_vid"][0] == 1 and d["leader_hops"][0] == g["expect_hops_K2"]
        a = idm_closed(v, g["expect_gap"], v - vf)
    else:
        assert d["leader_vid"][0] == -1 and d["leader_hops"][0] == g["expect_hops_K1"]
        a = idm_closed(v, 0.0, 0.0, lead=False)
    assert close(d["accel"][0], a), (d["accel"][0], a)
    assert close(r.state()["s"][0], g["ego"][0] + (v + (v + a)) / 2.0)


@pytest.mark.parametrize("exact", MODES)
def test_stop_within_step_gpu(simlib, exact):
    g = GOLD["STOP-IN-STEP"]
    r = Run(simlib, PS.stop_in_step(tuple(g["ego"]), tuple(g["lead"])), 1, exact)
    assert r.dec()["accel"][0] == g["expect_a"]
    st = r.state()
    assert st["s"][0] == g["expect_s"] and st["v"][0] == g["expect_v"]


@pytest.mark.parametrize("exact", MODES)
def test_two_lane_crossing_in_one_step_gpu(simlib, exact):
    g = GOLD["CROSS-TWO"]
    s, v = g["ego"]
    scen, (a0, j, b0) = PS.crossing(tuple(g["ego"]), g["L_j"])
    r = Run(simlib, scen, 1, exact)
    st, d = r.state(), r.dec()
    a = idm_closed(v, 0.0, 0.0, lead=False)
    s1 = ((s + (v + (v + a)) / 2.0) - 100.0) - g["L_j"]
    assert d["handoffs"][0] == g["expect_handoffs"]
    assert st["lane"][0] == b0 and st["cursor"][0] == g["expect_cursor"]
    assert close(st["s"][0], s1)
