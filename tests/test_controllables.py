"""Remaining controllable objects and metrics (Table 1
P:1074-1082, §3.2): set_tl_policy, set_lane_max_speed,
set_lane_restriction, set_tl_duration, road travelling speed.
Readings L42-L45.

Oracle pins (CPU):
  * NONE policy -> every junction lane GREEN;
  * a lane speed change moves the free-road equilibrium speed to the new
    v0 = min(lane, vehicle) (IDM closed form: a = 0 iff v = v0);
  * restricting the only exit lane makes approaching vehicles queue at the
    road end; lifting it releases them;
  * switching FIXED_TIME -> MAX_PRESSURE restarts the green timer (L42);
  * set_tl_duration holds the current green d steps, then yellow, then the
    next phase (L43), signal by signal;
  * road average speed = brute-force mean of the vehicle speeds on the road's
    lanes, the road's max lane speed when it is empty (L45).
GPU: the same setter sequences bit-identical to the oracle in exact mode, and
road speeds within the fp tolerance.
"""
import numpy as np
import pytest

import synth

SIG_GREEN = 0
POL_NONE, POL_FIXED, POL_MANUAL, POL_MAXP = 0, 1, 2, 3


def test_none_policy_all_green(oracle_lib):
    sc = synth.grid(rows=2, cols=2, road_len=200.0, lanes=2, n_trips=100, seed=5)
    o = oracle_lib.Oracle(sc)
    for j in range(o.n_junctions):
        assert o.set_signal_policy(j, POL_NONE) == 0
    o.step(1)
    st = o.read_state()
    jl = sc.graph["junc_lanes"]
    assert np.all(st["lane_signal"][jl] == SIG_GREEN)
    assert np.all(st["junc_policy"] == POL_NONE)


def synth_oracle():
    import oracle
    return oracle.Oracle(synth.grid(rows=2, cols=2, road_len=200.0, lanes=2, n_trips=50, seed=8))


def _one_lane(length=2000.0, vmax=13.9, n=1):
    b = synth.NetBuilder()
    r = b.add_road(1, length, vmax)
    lane = b.road_lanes[r][0]
    trips = dict(depart_step=np.zeros(n, np.int32), on_network_at_t0=np.ones(n, np.uint8),
                 route_offsets=np.arange(n + 1, dtype=np.int32), route_roads=np.full(n, r, np.int32),
                 start_lane=np.full(n, lane, np.int32),
                 start_s=np.array([10.0 + 20 * k for k in range(n)], np.float32),
                 start_v=np.zeros(n, np.float32), end_s=np.full(n, length, np.float32),
                 profile=np.zeros(n, np.uint8))
    return synth.Scenario("lane", b.graph(), trips, synth.default_profiles(),
                          synth.default_params(1)), lane


def test_lane_max_speed_sets_free_flow(oracle_lib):
    sc, lane = _one_lane()
    o = oracle_lib.Oracle(sc)
    o.step(60)
    assert abs(o.read_state()["v"][0] - 13.9) < 1e-3          # v0 = min(13.9, 16.667)
    assert o.set_lane_max_speed(lane, 8.0) == 0
    o.step(1)
    a = o.decisions()["accel"][0]
    x = o.read_state()["v"][0]
    assert a < -1.0                                            # IDM free term 2(1-(13.9/8)^4) < 0
    o.step(80)
    assert abs(o.read_state()["v"][0] - 8.0) < 1e-3
    assert o.set_lane_max_speed(lane, 0.0) != 0                # rejected


def test_restriction_queues_and_releases(oracle_lib):
    sc, jls = synth.pressure_junction([4, 0, 0, 0, 0, 0], period=30)
    g = sc.graph
    o = oracle_lib.Oracle(sc)
    for j in range(o.n_junctions):
        o.set_signal_policy(j, POL_NONE)                       # no signal: only the restriction stops them
    exit_lane = int(g["succ_lanes"][g["succ_offsets"][jls[0]]])
    o.set_lane_restriction(exit_lane, 1)
    o.step(120)
    st = o.read_state()
    a_lane = int(g["road_lanes"][0])
    assert np.all(st["lane"] == a_lane) and np.all(st["status"] == 1)
    assert np.all(st["s"] <= g["lane_length"][a_lane] + 1e-9)
    assert np.all(st["v"] < 0.1)                               # queued at the road end
    o.set_lane_restriction(exit_lane, 0)
    o.step(120)
    assert np.all(o.read_state()["status"] == 2)               # released, all arrived


def test_policy_switch_restarts_timer(oracle_lib):
    sc = synth.grid(rows=2, cols=2, road_len=200.0, lanes=2, n_trips=200, seed=6)
    o = oracle_lib.Oracle(sc)
    o.step(17)
    o.set_signal_policy(0, POL_MAXP)
    o.step(1)
    st = o.read_state()
    assert st["junc_policy"][0] == POL_MAXP
    # timer restarted at the switch, then advanced once by this step
    assert st["junc_elapsed"][0] == 1 or st["junc_yellow_left"][0] > 0


def _duration_timeline(sim, sc, t0, d, n_steps):
    """Per step: (phase of the green / yellow seen by vehicles) for junction 0."""
    g = sc.graph
    lanes = g["junc_lanes"][g["junc_lane_offsets"][0]:g["junc_lane_offsets"][1]]
    sim.step(t0)
    st = sim.read_state()
    p0, y0 = int(st["junc_phase"][0]), int(st["junc_yellow_left"][0])
    sim.set_signal_duration(0, d)
    out = []
    for _ in range(n_steps):
        sim.step(1)
        st = sim.read_state()
        out.append(tuple(int(x) for x in st["lane_signal"][lanes]))
    return p0, y0, out, st


def test_signal_duration_holds_then_advances(oracle_lib):
    """set_tl_duration: the current green is held d steps, then
    the yellow (Y = 3) and the next phase."""
    sc = synth.grid(rows=2, cols=2, road_len=200.0, lanes=2, n_trips=50, seed=8)
    o = oracle_lib.Oracle(sc)
    p0, y0, tl, st = _duration_timeline(o, sc, 40, 5, 10)
    g = sc.graph
    K = g["junc_phase_offsets"][1] - g["junc_phase_offsets"][0]
    ns = g["junc_lane_offsets"][1] - g["junc_lane_offsets"][0]
    green = g["phase_green"][:K * ns].reshape(K, ns)
    assert y0 == 0                                             # called during a green
    exp_p = tuple(0 if green[p0][k] else 2 for k in range(ns))
    exp_y = tuple(1 if green[p0][k] else 2 for k in range(ns))
    exp_n = tuple(0 if green[(p0 + 1) % K][k] else 2 for k in range(ns))
    assert tl[:5] == [exp_p] * 5, tl
    assert tl[5:8] == [exp_y] * 3, tl
    assert tl[8:] == [exp_n] * 2, tl
    assert st["junc_policy"][0] == POL_MANUAL and st["junc_remaining"][0] == -1


def test_road_avg_speed_brute_force(oracle_lib):
    sc = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=900, seed=7)
    g = sc.graph
    o = oracle_lib.Oracle(sc)
    o.step(200)
    st = o.read_state()
    got = o.road_avg_speed()
    nr = len(g["road_lane_offsets"]) - 1
    for r in range(nr):
        lanes = g["road_lanes"][g["road_lane_offsets"][r]:g["road_lane_offsets"][r + 1]]
        on = (st["status"] == 1) & np.isin(st["lane"], lanes)
        exp = st["v"][on].mean() if on.any() else g["lane_max_speed"][lanes].max()
        assert abs(got[r] - exp) <= 1e-12 * max(1.0, abs(exp)), r


def _setter_script(sc, rng, n_rounds):
    """Random sequence of (kind, args) setter calls between 25-step chunks."""
    g = sc.graph
    nj = len(g["junc_lane_offsets"]) - 1
    road_lanes = np.where(g["lane_road"] >= 0)[0]
    out = []
    for _ in range(n_rounds):
        calls = []
        for j in rng.choice(nj, 2, replace=False):
            calls.append(("policy", int(j), int(rng.choice([POL_NONE, POL_FIXED, POL_MANUAL, POL_MAXP]))))
        for l in rng.choice(road_lanes, 3, replace=False):
            calls.append(("speed", int(l), float(rng.choice([6.0, 10.0, 16.667]))))
        for l in rng.choice(len(g["lane_length"]), 2, replace=False):
            calls.append(("restrict", int(l), int(rng.integers(2))))
        calls.append(("duration", int(rng.integers(nj)), int(rng.integers(1, 12))))
        out.append(calls)
    return out


def _apply(sim, calls):
    for kind, a, b in calls:
        if kind == "policy":
            sim.set_signal_policy(a, b)
        elif kind == "speed":
            sim.set_lane_max_speed(a, b)
        elif kind == "duration":
            sim.set_signal_duration(a, b)
        else:
            sim.set_lane_restriction(a, b)


@pytest.mark.gpu
def test_setters_exact_mode_bit_identical(oracle_lib):
    import paper_2406_10661_b200 as p
    p.build()
    sc = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=81)
    g = p.Sim.from_scenario(sc, exact_mode=True)
    o = oracle_lib.Oracle(sc, store_fp32=True)
    for rnd, calls in enumerate(_setter_script(sc, np.random.default_rng(3), 8)):
        _apply(g, calls)
        _apply(o, calls)
        g.step(25)
        o.step(25)
        gs, os_ = g.read_state(), o.read_state()
        for k in ("status", "lane", "cursor", "wait_steps", "junc_policy", "junc_phase",
                  "junc_elapsed", "junc_yellow_left", "junc_remaining", "lane_signal"):
            assert np.array_equal(gs[k], os_[k]), (rnd, k)
        d = os_["status"] == 1
        assert np.array_equal(gs["s"][d].astype(np.float64), os_["s"][d]), rnd
        rs = g.read_metrics(road_speed=True)["road_avg_speed"]
        ro = o.road_avg_speed()
        assert np.all(np.abs(rs - ro) <= 1e-5 * np.maximum(1.0, np.abs(ro))), rnd


@pytest.mark.gpu
def test_setter_pins_gpu():
    import paper_2406_10661_b200 as p
    p.build()
    sc = synth.grid(rows=2, cols=2, road_len=200.0, lanes=2, n_trips=50, seed=8)
    o_tl = _duration_timeline(synth_oracle(), sc, 40, 5, 10)
    g_tl = _duration_timeline(p.Sim.from_scenario(sc), sc, 40, 5, 10)
    assert o_tl[2] == g_tl[2]
    sc, lane = _one_lane()
    g = p.Sim.from_scenario(sc)
    g.step(60)
    g.set_lane_max_speed(lane, 8.0)
    g.step(81)
    assert abs(g.read_state()["v"][0] - 8.0) < 1e-3
    sc, jls = synth.pressure_junction([4, 0, 0, 0, 0, 0], period=30)
    gr = sc.graph
    g = p.Sim.from_scenario(sc)
    g.set_signal_policy(0, POL_NONE)
    ex = int(gr["succ_lanes"][gr["succ_offsets"][jls[0]]])
    g.set_lane_restriction(ex, 1)
    g.step(120)
    st = g.read_state()
    assert np.all(st["status"] == 1) and np.all(st["v"] < 0.1)
    assert np.all(st["lane_signal"][gr["junc_lanes"]] == SIG_GREEN)
    g.set_lane_restriction(ex, 0)
    g.step(120)
    assert np.all(g.read_state()["status"] == 2)


def _road_adj(g):
    adj = {}
    lr = g["lane_road"]
    for l in np.where(lr >= 0)[0]:
        for e in range(g["succ_offsets"][l], g["succ_offsets"][l + 1]):
            j = g["succ_lanes"][e]
            t = lr[j] if lr[j] >= 0 else lr[g["succ_lanes"][g["succ_offsets"][j]]]
            adj.setdefault(int(lr[l]), set()).add(int(t))
    return {k: sorted(v) for k, v in adj.items()}


def _walk(adj, start, n, rng, second=None):
    r = [start] + ([second] if second is not None else [])
    while len(r) < n and adj.get(r[-1]):
        r.append(int(rng.choice(adj[r[-1]])))
    return r


def _reroutes(sc, st, rng, k_driving=20, k_pending=10):
    """Valid new routes for random DRIVING / PENDING vehicles of state st."""
    g, tr = sc.graph, sc.trips
    adj = _road_adj(g)
    lr = g["lane_road"]
    out = []
    cur_road = lambda k: int(tr["route_roads"][tr["route_offsets"][k]])
    drv = np.where(st["status"] == 1)[0]
    pen = np.where(st["status"] == 0)[0]
    for k in rng.choice(drv, min(k_driving, len(drv)), replace=False):
        lane = int(st["lane"][k])
        if lr[lane] < 0:
            continue                                   # junction lanes: covered by the GPU test's rule
        r = _walk(adj, int(lr[lane]), 4, rng)
        out.append((int(k), r, float(g["lane_length"][g["road_lanes"][g["road_lane_offsets"][r[-1]]]])))
    for k in rng.choice(pen, min(k_pending, len(pen)), replace=False):
        r = _walk(adj, cur_road(int(k)), 5, rng)
        out.append((int(k), r, 10.0))
    return out


def test_vehicle_route_pins(oracle_lib):
    """set_vehicle_route: after the change the vehicle travels the
    new route's roads in order and arrives at its end; invalid
    requests change nothing."""
    sc = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=600, seed=9)
    g = sc.graph
    o = oracle_lib.Oracle(sc)
    o.step(150)
    st = o.read_state()
    rng = np.random.default_rng(4)
    lr = g["lane_road"]
    adj = _road_adj(g)
    k = next(int(k) for k in np.where(st["status"] == 1)[0] if lr[st["lane"][k]] >= 0)
    r = _walk(adj, int(lr[st["lane"][k]]), 4, rng)
    end = float(g["lane_length"][g["road_lanes"][g["road_lane_offsets"][r[-1]]]])
    bad = [x for x in range(len(g["road_lane_offsets"]) - 1) if x != r[0]][0]
    assert o.set_vehicle_route(k, [bad] + r[1:], end) != 0       # must start on the current road
    assert o.set_vehicle_route(k, r, end) == 0
    seen = []
    for _ in range(1500):
        o.step(1)
        s2 = o.read_state()
        if s2["status"][k] == 2:
            break
        rd = int(lr[s2["lane"][k]])
        if rd >= 0 and (not seen or seen[-1] != rd):
            seen.append(rd)
    assert s2["status"][k] == 2
    assert seen == r[:len(seen)] and seen[-1] == r[-1], (seen, r)
    assert o.set_vehicle_route(k, r, end) != 0                    # finished


@pytest.mark.gpu
def test_vehicle_route_exact_mode_bit_identical(oracle_lib):
    import paper_2406_10661_b200 as p
    p.build()
    sc = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=82)
    gsim = p.Sim.from_scenario(sc, exact_mode=True)
    o = oracle_lib.Oracle(sc, store_fp32=True)
    rng = np.random.default_rng(5)
    for rnd in range(6):
        gsim.step(40)
        o.step(40)
        req = _reroutes(sc, o.read_state(), rng)
        for k, r, e in req:
            assert o.set_vehicle_route(k, r, e) == 0
        gsim.set_vehicle_route_batch([k for k, _, _ in req], [r for _, r, _ in req],
                                     [e for _, _, e in req])
        gs, os_ = gsim.read_state(), o.read_state()
        for key in ("status", "lane", "cursor"):
            assert np.array_equal(gs[key], os_[key]), (rnd, key)
    gsim.step(300)
    o.step(300)
    gs, os_ = gsim.read_state(), o.read_state()
    for key in ("status", "lane", "cursor", "wait_steps", "arrive_time"):
        assert np.array_equal(gs[key], os_[key]), key
    d = os_["status"] == 1
    assert np.array_equal(gs["s"][d].astype(np.float64), os_["s"][d])
