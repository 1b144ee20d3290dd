"""Direct evidence for the per-lane ordering (row a1, P:130, P:803-807;
VERDICT r01 "Next round" #2a/#2b).

The step kernel keeps each road tile's vehicles as sorted stayers plus an
unsorted inbox and merges the two at the start of every step.  Here states
are loaded with a chosen share of the DRIVING vehicles placed in the inboxes
(sim_load_state_inbox), including equal-s ties with stayers (synth
random_state ties, ledger L12) and tiles with hundreds of inbox records, and:
  * the lane order sim_read_state reports is the kernel's own merge of those
    records (k_lane_order), compared with the oracle's (s, vid) sort of the
    same state — identical, element by element (after a step, positions
    carry fp32 rounding, so orders may differ only between near-equal s);
  * one step from that state matches the oracle like the empty-inbox battery
    of test_gpu_parity.py (integer outputs exact, s / v / a within 1e-5).
"""
import numpy as np
import pytest

import synth
from parity import compare_decisions, compare_lane_orders, compare_states

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def simlib():
    import paper_2406_10661_b200 as p
    p.build()
    return p


SCENARIOS = {
    "grid2": lambda: synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=21),
    "grid3_tidal_dyn": lambda: synth.grid(rows=3, cols=3, road_len=250.0, lanes=3, n_trips=2000,
                                          seed=22, tidal=True, dynamic=True),
    "ring3": lambda: synth.ring(n_vehicles=120, n_lanes=3, length=800.0, seed=24),
    "city": lambda: synth.city(G=8, n_vehicles=6000, seed=25),
}


def _load_pair(simlib, oracle_lib, scen, st, to_inbox, exact=False):
    g = simlib.Sim.from_scenario(scen, exact_mode=exact, record_decisions=True)
    o = oracle_lib.Oracle(scen)
    g.load_state(st, to_inbox=to_inbox)
    o.load_state({k: (v.astype(np.float64) if k in ("s", "v") else v) for k, v in st.items()})
    return g, o


def _assert_same_order(g, o):
    gs = g.read_state(lane_order=True)
    o_off, o_ord = o.lane_order()
    assert np.array_equal(gs["lane_offsets"], o_off)
    bad = np.where(gs["lane_order"] != o_ord)[0]
    assert bad.size == 0, f"lane order differs at {bad[:10]}: gpu {gs['lane_order'][bad[:5]]} oracle {o_ord[bad[:5]]}"


@pytest.mark.parametrize("frac", [0.35, 1.0])
@pytest.mark.parametrize("name", list(SCENARIOS))
def test_merge_order_and_step_with_populated_inboxes(simlib, oracle_lib, name, frac):
    scen = SCENARIOS[name]()
    for seed in range(3):
        st = synth.random_state(scen, seed=300 + seed)
        rng = np.random.default_rng(seed)
        to_inbox = ((st["status"] == 1) & (rng.random(scen.n_trips) < frac)).astype(np.uint8)
        g, o = _load_pair(simlib, oracle_lib, scen, st, to_inbox)
        _assert_same_order(g, o)                        # the merge (a1), before any step
        g.step(1)
        o.step(1)
        where = f"[{name} frac={frac} seed={seed}] "
        compare_decisions(g.read_decisions(), o.decisions(), st["status"], where=where)
        gs = g.read_state(lane_order=True)
        compare_states(gs, o.read_state(), where=where)
        o_off, o_ord = o.lane_order()                    # after the step: equal up to fp near-ties
        compare_lane_orders(gs["lane_offsets"], gs["lane_order"], o_off, o_ord, gs)


def _long_road(n_veh, n_lanes=3, L=3000.0, seed=5):
    """One long multi-lane road: a single tile holding n_veh vehicles (more than
    the shared-memory ring takes: the tile runs in global mode)."""
    b = synth.NetBuilder()
    r = b.add_road(n_lanes, L, 16.667)
    rng = np.random.default_rng(seed)
    lanes = rng.integers(0, n_lanes, n_veh)
    s = np.sort(rng.random(n_veh)) * (L - 100.0) + 20.0
    s = s.astype(np.float32)
    s[1::7] = s[0::7][:len(s[1::7])]                    # equal-s ties across lanes and records
    trips = dict(depart_step=np.zeros(n_veh, np.int32), on_network_at_t0=np.ones(n_veh, np.uint8),
                 route_offsets=np.arange(n_veh + 1).astype(np.int32), route_roads=np.zeros(n_veh, np.int32),
                 start_lane=np.array([b.road_lanes[r][x] for x in lanes], np.int32), start_s=s,
                 start_v=(rng.random(n_veh) * 12).astype(np.float32),
                 end_s=np.full(n_veh, L, np.float32), profile=np.zeros(n_veh, np.uint8))
    return synth.Scenario("long", b.graph(), trips, synth.default_profiles(), synth.default_params(9))


@pytest.mark.parametrize("n_veh,frac", [(300, 0.4), (1500, 0.2)])
def test_large_inbox_and_global_mode_tile(simlib, oracle_lib, n_veh, frac):
    """A tile with 120 / 300 inbox records (the round-1 kernel sorted at most
    48 in shared memory); 1500 vehicles exceed the ring slot, so that tile
    runs the global-mode instantiation."""
    scen = _long_road(n_veh)
    o0 = oracle_lib.Oracle(scen)
    st = o0.read_state()
    st["s"] = st["s"].astype(np.float32)
    st["v"] = st["v"].astype(np.float32)
    rng = np.random.default_rng(n_veh)
    to_inbox = ((st["status"] == 1) & (rng.random(scen.n_trips) < frac)).astype(np.uint8)
    assert to_inbox.sum() > 48
    # fp32 path: one step against the fp64 oracle (tolerance of SURVEY 8(c).4)
    g, o = _load_pair(simlib, oracle_lib, scen, st, to_inbox)
    _assert_same_order(g, o)
    g.step(1)
    o.step(1)
    compare_decisions(g.read_decisions(), o.decisions(), st["status"], where=f"[long {n_veh}] ")
    compare_states(g.read_state(), o.read_state(), where=f"[long {n_veh}] ")
    # exact mode: several steps, bit-identical to the oracle with fp32 storage (P-EXACT)
    g = simlib.Sim.from_scenario(scen, exact_mode=True)
    o = oracle_lib.Oracle(scen, store_fp32=True)
    g.load_state(st, to_inbox=to_inbox)
    o.load_state({k: (v.astype(np.float64) if k in ("s", "v") else v) for k, v in st.items()})
    g.step(4)
    o.step(4)
    gs, os_ = g.read_state(), o.read_state()
    for k in ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time"):
        assert np.array_equal(gs[k], os_[k]), k
    d = os_["status"] == 1
    assert np.array_equal(gs["s"][d].astype(np.float64), os_["s"][d])
    assert np.array_equal(gs["v"][d].astype(np.float64), os_["v"][d])
