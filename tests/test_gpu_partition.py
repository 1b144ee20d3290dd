"""P-PART on one GPU: the partitioned path (spatial partition of road tiles,
migration of boundary vehicles, halo of lane summaries) run with
the loopback transport gives bit-identical state and metrics for any number
of partitions — decisions depend only on the snapshot and (seed, vid, t), and
every reduction is integer.  direct=True is the NEXT-2
transport: the step kernel writes movers and summaries straight
into the owning partition's buffers, with no exchange step."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def simlib():
    import paper_2406_10661_b200 as p
    p.build()
    return p


def _run(simlib, scen, steps, **kw):
    g = simlib.Sim.from_scenario(scen, **kw)
    g.step(steps)
    return g.read_state(lane_order=True), g.read_metrics(lane_stats=True)


KEYS = ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v",
        "lane_offsets", "lane_order")
MKEYS = ("n_pending", "n_driving", "n_finished", "vehicle_steps", "sum_travel_steps",
         "sum_wait_steps_finished", "sum_depart_delay", "n_lane_changes", "n_handoffs",
         "n_inserted", "n_guard_hits")


@pytest.mark.parametrize("direct", [False, True])
@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("name", ["grid", "city", "grid_maxpressure"])
def test_partition_invariance(simlib, name, world, direct):
    """grid_maxpressure: the MAX_PRESSURE choice needs every lane's count, so
    the partitions' counts must add up exactly (shared buffer / allreduce)."""
    if name == "city":
        scen = synth.city(G=12, n_vehicles=20000, seed=13)
    else:
        scen = synth.grid(rows=4, cols=4, road_len=250.0, lanes=2, n_trips=3000, seed=12,
                          depart_window=400,
                          policy=synth.POLICY_MAXP if name == "grid_maxpressure" else synth.POLICY_FIXED)
    s1, m1 = _run(simlib, scen, 150)
    sw, mw = _run(simlib, scen, 150, world=world, loopback=True, direct=direct)
    for k in KEYS:
        assert np.array_equal(s1[k], sw[k]), (k, world)
    for k in MKEYS:
        assert m1[k] == mw[k], (k, world, m1[k], mw[k])
    assert np.array_equal(m1["lane_count"], mw["lane_count"])
    assert np.array_equal(m1["lane_waiting_at_end"], mw["lane_waiting_at_end"])
    assert m1["n_handoffs"] > 0


@pytest.mark.parametrize("direct", [False, True])
def test_partitioned_exact_mode_matches_oracle(simlib, oracle_lib, direct):
    """The partitioned path is still the model: exact mode with 3 partitions
    equals the oracle (store_fp32) bit for bit."""
    scen = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=21)
    g = simlib.Sim.from_scenario(scen, exact_mode=True, world=3, loopback=True, direct=direct)
    o = oracle_lib.Oracle(scen, store_fp32=True)
    g.step(200)
    o.step(200)
    gs, os_ = g.read_state(), o.read_state()
    for k in ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time"):
        assert np.array_equal(gs[k], os_[k]), k
    d = os_["status"] == 1
    assert np.array_equal(gs["s"][d].astype(np.float64), os_["s"][d])


@pytest.mark.parametrize("direct", [False, True])
def test_partitioned_decisions_and_setters(simlib, direct):
    scen = synth.grid(rows=3, cols=3, road_len=250.0, lanes=3, n_trips=1500, seed=31,
                      tidal=True, dynamic=True, depart_window=300)
    a = simlib.Sim.from_scenario(scen, record_decisions=True)
    b = simlib.Sim.from_scenario(scen, record_decisions=True, world=4, loopback=True,
                                 direct=direct)
    rng = np.random.default_rng(1)
    dyn = np.where(scen.graph["lane_kind"] == 1)[0]
    for t in range(6):
        ls = dyn[rng.random(len(dyn)) < 0.4]
        ds = rng.integers(0, 2, len(ls))
        js = rng.choice(len(scen.graph["junc_lane_offsets"]) - 1, 2, replace=False)
        ps = rng.integers(0, 4, 2)
        for sim in (a, b):
            sim.set_lane_direction_batch(ls, ds)
            sim.set_signal_phase_batch(js, ps)
            sim.step(25)
        da, db = a.read_decisions(), b.read_decisions()
        for k in ("leader_vid", "lc", "handoffs", "inserted", "finished", "side_vid"):
            assert np.array_equal(da[k], db[k]), (t, k)
        sa, sb = a.read_state(), b.read_state()
        for k in ("status", "lane", "s", "v", "junc_phase", "lane_signal"):
            assert np.array_equal(sa[k], sb[k]), (t, k)


@pytest.mark.parametrize("name", ["city", "grid_maxpressure"])
def test_repartition_invariance(simlib, name):
    """NEXT-2 dynamic repartitioning: tiles handed to new owners
    at step boundaries (an explicit scattered partition, then the library's
    load rebalance) leave every result bit-identical to one partition."""
    if name == "city":
        scen = synth.city(G=12, n_vehicles=20000, seed=13)
    else:
        scen = synth.grid(rows=4, cols=4, road_len=250.0, lanes=2, n_trips=3000, seed=12,
                          depart_window=400, policy=synth.POLICY_MAXP)
    world = 3
    a = simlib.Sim.from_scenario(scen)
    b = simlib.Sim.from_scenario(scen, world=world, loopback=True, direct=True)
    nr = len(scen.graph["road_lane_offsets"]) - 1
    for sim in (a, b):
        sim.step(60)
    assert b.repartition((np.arange(nr) * 7) % world) > 0
    for sim in (a, b):
        sim.step(60)
    b.repartition()
    assert b.repartition() == 0                    # balanced already: nothing moves
    for sim in (a, b):
        sim.step(40)
    s1, m1 = a.read_state(lane_order=True), a.read_metrics(lane_stats=True)
    sw, mw = b.read_state(lane_order=True), b.read_metrics(lane_stats=True)
    for k in KEYS:
        assert np.array_equal(s1[k], sw[k]), k
    for k in MKEYS:
        assert m1[k] == mw[k], (k, m1[k], mw[k])
    assert np.array_equal(m1["lane_count"], mw["lane_count"])


def test_repartition_needs_direct_transport(simlib):
    scen = synth.grid(rows=2, cols=2, road_len=200.0, lanes=1, n_trips=50, seed=3)
    g = simlib.Sim.from_scenario(scen, world=2, loopback=True)
    with pytest.raises(simlib.SimError) as e:
        g.repartition()
    assert e.value.status == 1                     # SIM_E_INVALID


def test_full_size_c4_direct_partitions(simlib):
    """BASELINE.json configs[3] at full size (C4, 2M vehicles): 8 partitions
    (the recursive coordinate bisection bench.py uses) with the direct
    transport, a load rebalance half way, against one partition — bit for bit."""
    scen = synth.city()
    a = simlib.Sim.from_scenario(scen)
    b = simlib.Sim.from_scenario(scen, world=8, loopback=True, direct=True,
                                 road_owner=synth.rcb_partition(scen, 8))
    for sim in (a, b):
        sim.step(20)
    assert b.repartition() > 0
    for sim in (a, b):
        sim.step(10)
    s1, sw = a.read_state(), b.read_state()
    for k in ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v"):
        assert np.array_equal(s1[k], sw[k]), k
    m1, mw = a.read_metrics(), b.read_metrics()
    for k in MKEYS:
        assert m1[k] == mw[k], (k, m1[k], mw[k])
    assert m1["n_handoffs"] > 50_000


def test_repartition_metrics_every_step(simlib):
    """after sim_repartition the old owner must not keep a
    stale stayer count of a moved tile in its other-parity buffer; reads on
    odd and even steps after the move equal one partition."""
    scen = synth.grid(rows=4, cols=4, road_len=250.0, lanes=2, n_trips=3000, seed=12, depart_window=400)
    world = 3
    a = simlib.Sim.from_scenario(scen)
    b = simlib.Sim.from_scenario(scen, world=world, loopback=True, direct=True)
    nr = len(scen.graph["road_lane_offsets"]) - 1
    for sim in (a, b):
        sim.step(41)
    assert b.repartition((np.arange(nr) * 5 + 1) % world) > 0
    for k in range(5):
        for sim in (a, b):
            sim.step(1)
        m1, mw = a.read_metrics(), b.read_metrics()
        for key in MKEYS:
            assert m1[key] == mw[key], (k, key, m1[key], mw[key])


def test_repartition_group_metrics(simlib):
    """per-group counters (batched environments) keep the rows a
    tile accumulated before it changed owner."""
    envs = [synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=800, seed=71),
            synth.grid(rows=3, cols=2, road_len=200.0, lanes=2, n_trips=700, seed=73)]
    B = synth.batch(envs)
    a = simlib.Sim.from_scenario(B)
    b = simlib.Sim.from_scenario(B, world=2, loopback=True, direct=True)
    nr = len(B.graph["road_lane_offsets"]) - 1
    for sim in (a, b):
        sim.step(80)
    assert b.repartition((np.arange(nr) * 3) % 2) > 0
    for sim in (a, b):
        sim.step(57)
    ga, gb = a.read_group_metrics(len(envs)), b.read_group_metrics(len(envs))
    for e in range(len(envs)):
        for key in MKEYS:
            assert ga[e][key] == gb[e][key], (e, key, ga[e][key], gb[e][key])


def test_load_state_after_repartition(simlib):
    """the finished-count baseline of a load uses the same
    reduction as the reads (all tiles of all partitions), so n_finished stays
    right after a load that follows a repartition."""
    scen = synth.grid(rows=4, cols=4, road_len=250.0, lanes=2, n_trips=3000, seed=12, depart_window=400)
    a = simlib.Sim.from_scenario(scen)
    b = simlib.Sim.from_scenario(scen, world=3, loopback=True, direct=True)
    nr = len(scen.graph["road_lane_offsets"]) - 1
    for sim in (a, b):
        sim.step(300)
    assert b.repartition((np.arange(nr) * 2) % 3) > 0
    for sim in (a, b):
        sim.step(101)
    st = a.read_state()
    for sim in (a, b):
        sim.load_state(st)
        sim.step(33)
    m1, mw = a.read_metrics(), b.read_metrics()
    assert m1["n_finished"] > 0
    for key in ("n_pending", "n_driving", "n_finished"):
        assert m1[key] == mw[key], (key, m1[key], mw[key])
