"""Step graphs: sim_step(n >= 12) replays a captured CUDA graph
of 6 steps whose kernels are chained by programmatic dependent launches.
The result must be bit-identical to stepping one launch at a time, for any
starting t mod 6, across host-side changes between calls (re-capture), with
MAX_PRESSURE lane counts, decision recording and loopback partitions."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

KEYS = ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v",
        "junc_phase", "junc_elapsed", "junc_yellow_left")


@pytest.fixture(scope="module")
def simlib():
    import paper_2406_10661_b200 as p
    p.build()
    return p


def _same(a, b, where=""):
    sa, sb = a.read_state(), b.read_state()
    for k in KEYS:
        assert np.array_equal(sa[k], sb[k]), where + k
    ma, mb = a.read_metrics(), b.read_metrics()
    for k in ("t", "n_driving", "n_finished", "vehicle_steps", "n_lane_changes", "n_handoffs",
              "n_inserted", "sum_travel_steps", "sum_depart_delay"):
        assert ma[k] == mb[k], where + k


def _eager(b, n):
    for _ in range(n):
        b.step(1)


@pytest.mark.parametrize("name", ["grid", "maxp", "city"])
def test_graph_replay_bit_identical(simlib, name):
    scen = {"grid": lambda: synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=31),
            "maxp": lambda: synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=32,
                                       policy=synth.POLICY_MAXP),
            "city": lambda: synth.city(G=8, n_vehicles=6000, seed=33)}[name]()
    a = simlib.Sim.from_scenario(scen, step_graphs=True)
    b = simlib.Sim.from_scenario(scen, step_graphs=False)
    # start at t = 0, then at t = 3 (another phase of the 6-step buffer period)
    a.step(60); _eager(b, 60)
    _same(a, b, f"[{name} t=60] ")
    a.step(3); b.step(3)
    a.step(31); _eager(b, 31)                       # 5 replays + 1 eager step
    _same(a, b, f"[{name} t=94] ")


def test_graph_recaptured_after_host_changes(simlib):
    scen = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=34)
    a = simlib.Sim.from_scenario(scen, step_graphs=True)
    b = simlib.Sim.from_scenario(scen, step_graphs=False)
    nj = a.n_junctions
    rng = np.random.default_rng(0)
    for it in range(4):
        a.step(24); _eager(b, 24)
        js = np.arange(nj, dtype=np.int32)
        ph = rng.integers(0, 2, nj).astype(np.int32)
        for s in (a, b):
            s.set_signal_phase_batch(js, ph)
            s.set_lane_max_speed(3, 8.0 + it)
            if it == 2:
                s.set_signal_policy(0, synth.POLICY_MAXP)    # MAX_PRESSURE appears: new launch args
    a.step(24); _eager(b, 24)
    _same(a, b, "[setters] ")
    # a state loaded mid-run (same t mod 6 and host arguments: the graph is reused)
    st = synth.random_state(scen, seed=5, t=a.read_metrics()["t"])
    a.load_state(st); b.load_state(st)
    a.step(18); _eager(b, 18)
    _same(a, b, "[load_state] ")


def test_graph_with_recording_and_partitions(simlib):
    scen = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=35)
    a = simlib.Sim.from_scenario(scen, step_graphs=True, record_decisions=True)
    b = simlib.Sim.from_scenario(scen, step_graphs=False, record_decisions=True)
    a.step(36); _eager(b, 36)
    _same(a, b, "[record] ")
    da, db = a.read_decisions(), b.read_decisions()
    for k in da:
        assert np.array_equal(da[k], db[k]), k
    for direct in (False, True):
        c = simlib.Sim.from_scenario(scen, world=3, loopback=True, direct=direct, step_graphs=True)
        d = simlib.Sim.from_scenario(scen, step_graphs=False)
        c.step(48); _eager(d, 48)
        _same(c, d, f"[loopback direct={direct}] ")

