"""Oracle invariants (P-CONS, P-ORD, P-SIGT, P-PERM, P-LEAD, P-ATT) on full
runs and random states.  Expected behaviour comes from the paper's semantic
statements (snapshot isolation P:784-790, in-lane order P:803, red/yellow stop
P:200, fixed-time program P:839, metrics P:875-883) and brute-force scans
written here, never from the oracle itself.
"""
import numpy as np
import pytest

import synth

SIG_GREEN, SIG_YELLOW, SIG_RED = 0, 1, 2


@pytest.fixture(scope="module")
def c2_small():
    return synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=900,
                      depart_window=600, seed=11)


def _lane_orders(st):
    order = {}
    for k in np.where(st["status"] == 1)[0]:
        order.setdefault(int(st["lane"][k]), []).append(int(k))
    for l in order:
        order[l].sort(key=lambda k: (st["s"][k], k))
    return order


def test_conservation_order_overlap_redlight(oracle_lib, c2_small):
    """P-CONS, P-ORD, non-negative gaps for stayers,
    red-light compliance."""
    sc = c2_small
    g = sc.graph
    L = g["lane_length"]
    plen = sc.profiles[sc.trips["profile"].astype(int), 5]
    is_junc = g["lane_road"] < 0
    o = oracle_lib.Oracle(sc)
    prev = o.read_state()
    n = sc.n_trips
    for t in range(700):
        o.step(1)
        st = o.read_state()
        d = o.decisions()
        m = o.metrics()
        assert m["n_pending"] + m["n_driving"] + m["n_finished"] == n
        assert (st["status"] == 1).sum() == m["n_driving"]
        # lane counts sum to driving
        c, _ = o.lane_stats()
        assert c.sum() == m["n_driving"]
        po, no = _lane_orders(prev), _lane_orders(st)
        for l, ks in no.items():
            stay = [k for k in ks if prev["status"][k] == 1 and prev["lane"][k] == l]
            before = [k for k in po.get(l, []) if k in set(stay)]
            assert stay == before, "stayers overtook within a lane"
            for a, b in zip(ks, ks[1:]):
                if a in set(stay) and b in set(stay):
                    gp = (prev["s"][b] - prev["s"][a]) - plen[b]
                    gn = (st["s"][b] - st["s"][a]) - plen[b]
                    if gp >= 0:
                        assert gn >= -1e-9
        # red-light compliance: entering a junction lane needs GREEN at step t
        for k in np.where((prev["status"] == 1) & (st["status"] >= 1))[0]:
            l0 = prev["lane"][k]
            if is_junc[l0] or d["handoffs"][k] == 0:
                continue
            # first lane entered is the road lane's next lane: a junction lane here
            l1 = st["lane"][k] if st["status"][k] == 1 else -1
            if l1 >= 0 and is_junc[l1] and d["handoffs"][k] == 1:
                assert st["lane_signal"][l1] == SIG_GREEN
        # positions within lanes
        drv = st["status"] == 1
        assert np.all(st["s"][drv] >= 0)
        assert np.all(st["s"][drv] <= L[st["lane"][drv]] + 1e-9)
        assert np.all(st["v"][drv] >= 0)
        prev = st


def _closed_form_signal(t, green_steps, Y):
    """FIXED_TIME closed form: returns (phase, in_yellow)."""
    C = sum(g + Y for g in green_steps)
    tau = t % C
    acc = 0
    for k, gk in enumerate(green_steps):
        if tau < acc + gk:
            return k, False
        if tau < acc + gk + Y:
            return k, True
        acc += gk + Y
    raise AssertionError


def test_fixed_time_signal_cycle(oracle_lib):
    """P-SIGT: sig_t equals the closed form for every t; each lane is green
    g_k steps per cycle."""
    sc = synth.grid(rows=2, cols=2, road_len=200.0, lanes=2, n_trips=1, seed=3)
    g = sc.graph
    o = oracle_lib.Oracle(sc)
    Y = sc.params["yellow_steps"]
    nj = len(g["junc_lane_offsets"]) - 1
    green_count = np.zeros(sc.n_lanes, int)
    for t in range(2 * 102 + 7):
        o.step(1)
        sig = o.read_state()["lane_signal"]       # the sig_t vehicles saw in step t
        gi = 0
        for j in range(nj):
            lanes = g["junc_lanes"][g["junc_lane_offsets"][j]:g["junc_lane_offsets"][j + 1]]
            p0, p1 = g["junc_phase_offsets"][j], g["junc_phase_offsets"][j + 1]
            steps = list(g["phase_green_steps"][p0:p1])
            green = g["phase_green"][gi:gi + len(lanes) * (p1 - p0)].reshape(p1 - p0, len(lanes))
            gi += len(lanes) * (p1 - p0)
            k, yel = _closed_form_signal(t + int(g["junc_offset_steps"][j]), steps, Y)
            for s, l in enumerate(lanes):
                exp = (SIG_YELLOW if yel else SIG_GREEN) if green[k][s] else SIG_RED
                assert sig[l] == exp, (t, j, l)
                if t < 102:
                    green_count[l] += sig[l] == SIG_GREEN
    # NS straight lanes green 30 of 102 steps, NS left 15 (C2 program)
    jl = np.where(g["lane_road"] < 0)[0]
    assert set(np.unique(green_count[jl])) <= {30, 15}


def test_manual_phase_switch(oracle_lib):
    """MANUAL: a switch shows Y yellow steps of the old phase, then the
    new phase is green (ledger L21, L35)."""
    sc = synth.grid(rows=2, cols=2, road_len=200.0, lanes=1, n_trips=1, seed=3)
    g = sc.graph
    o = oracle_lib.Oracle(sc)
    o.step(5)                               # phase 0 green, no yellow yet
    lanes = g["junc_lanes"][g["junc_lane_offsets"][0]:g["junc_lane_offsets"][1]]
    nl = len(lanes)
    green = g["phase_green"][:4 * nl].reshape(4, nl)
    assert o.set_signal_phase(0, 2) == 0
    seen = []
    for _ in range(6):
        o.step(1)
        seen.append(o.read_state()["lane_signal"][lanes].copy())
    for t in range(3):
        exp = np.where(green[0] == 1, SIG_YELLOW, SIG_RED)
        assert np.array_equal(seen[t], exp)
    for t in range(3, 6):
        exp = np.where(green[2] == 1, SIG_GREEN, SIG_RED)
        assert np.array_equal(seen[t], exp)
    assert o.set_signal_phase(0, 99) != 0


def test_snapshot_isolation_reverse_order(oracle_lib, c2_small):
    """P-PERM: reversed processing order gives identical results."""
    a = oracle_lib.Oracle(c2_small)
    b = oracle_lib.Oracle(c2_small, reverse_order=True)
    a.step(300)
    b.step(300)
    sa, sb = a.read_state(), b.read_state()
    for k in ("status", "lane", "s", "v", "cursor", "wait_steps"):
        assert np.array_equal(sa[k], sb[k]), k
    assert a.metrics() == b.metrics()


def _brute_neighbours(st, k, lane_left, lane_right):
    """O(N^2) scans of the definitions."""
    key = lambda x: (st["s"][x], x)
    same = [x for x in np.where(st["status"] == 1)[0] if st["lane"][x] == st["lane"][k] and x != k]
    ahead = [x for x in same if key(x) > key(k)]
    behind = [x for x in same if key(x) < key(k)]
    lead = min(ahead, key=key) if ahead else -1
    of = max(behind, key=key) if behind else -1
    side = []
    for nb in (lane_left[st["lane"][k]], lane_right[st["lane"][k]]):
        if nb < 0:
            side += [-1, -1]
            continue
        on = [x for x in np.where(st["status"] == 1)[0] if st["lane"][x] == nb]
        fr = [x for x in on if st["s"][x] > st["s"][k]]
        bk = [x for x in on if st["s"][x] <= st["s"][k]]
        side += [min(fr, key=key) if fr else -1, max(bk, key=key) if bk else -1]
    return lead, of, side


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_leader_and_side_brute_force(oracle_lib, seed):
    """P-LEAD: in-lane leader / old follower / side neighbours equal an O(N^2)
    scan; a lookahead leader (hops >= 1) only when no in-lane leader exists and
    it is the first vehicle of its lane."""
    sc = synth.grid(rows=2, cols=2, road_len=150.0, lanes=2, n_trips=400, seed=5)
    st = synth.random_state(sc, seed=seed, t=40)
    o = oracle_lib.Oracle(sc)
    o.load_state(st)
    o.step(1)
    d = o.decisions()
    g = sc.graph
    for k in np.where(st["status"] == 1)[0]:
        lead, of, side = _brute_neighbours(st, k, g["lane_left"], g["lane_right"])
        if lead >= 0:
            assert d["leader_vid"][k] == lead and d["leader_hops"][k] == 0
        else:
            assert d["leader_hops"][k] != 0
            f = d["leader_vid"][k]
            if f >= 0:
                fl = st["lane"][f]
                firsts = [x for x in np.where(st["status"] == 1)[0] if st["lane"][x] == fl]
                assert f == min(firsts, key=lambda x: (st["s"][x], x))
        assert d["old_follower_vid"][k] == of
        if g["lane_road"][st["lane"][k]] >= 0:
            assert list(d["side_vid"][k]) == side


def test_metrics_consistency(oracle_lib, c2_small):
    """P-ATT: travel = arrive - insert summed over finished;
    ATT = sum / finished; TP = finished."""
    o = oracle_lib.Oracle(c2_small)
    o.step(800)
    st = o.read_state()
    m = o.metrics()
    fin = st["status"] == 2
    assert m["n_finished"] == fin.sum() > 0
    assert m["sum_travel_steps"] == int((st["arrive_time"][fin] - st["insert_time"][fin]).sum())
    assert m["att_finished"] == m["sum_travel_steps"] / m["n_finished"]
    ins = st["status"] >= 1
    assert m["sum_depart_delay"] == int((st["insert_time"][ins] -
                                         c2_small.trips["depart_step"][ins]).sum())


def test_determinism(oracle_lib, c2_small):
    a = oracle_lib.Oracle(c2_small)
    b = oracle_lib.Oracle(c2_small)
    a.step(200)
    b.step(200)
    assert a.metrics() == b.metrics()
    assert np.array_equal(a.read_state()["s"], b.read_state()["s"])


def test_dynamic_and_tidal_lanes(oracle_lib):
    """Dynamic lanes only feed the movement their direction
    enables; a disabled tidal lane takes no entries."""
    sc = synth.grid(rows=3, cols=3, road_len=300.0, lanes=3, n_trips=1500,
                    depart_window=600, seed=9, tidal=True, dynamic=True)
    g = sc.graph
    kinds, turn = g["lane_kind"], g["lane_turn"]
    succ_off, succ = g["succ_offsets"], g["succ_lanes"]
    pred = {}
    for l in range(sc.n_lanes):
        for j in succ[succ_off[l]:succ_off[l + 1]]:
            pred[int(j)] = l
    o = oracle_lib.Oracle(sc)
    dyn = np.where(kinds == 1)[0]
    tid = np.where(kinds == 2)[0]
    rng = np.random.default_rng(0)
    prev = o.read_state()
    dirs = g["lane_dir0"].copy()
    for t in range(600):
        if t % 30 == 0:
            for l in dyn:
                dnew = int(rng.integers(2))
                assert o.set_lane_direction(int(l), dnew) == 0
                dirs[l] = dnew
        if t % 180 == 0:
            for l in tid:
                if g["tidal_partner"][l] > l:
                    dnew = int(rng.integers(2))
                    o.set_lane_direction(int(l), dnew)
                    dirs[l], dirs[g["tidal_partner"][l]] = dnew, 1 - dnew
        o.step(1)
        st = o.read_state()
        moved = (prev["status"] == 1) & (st["status"] == 1) & (st["lane"] != prev["lane"])
        for k in np.where(moved)[0]:
            l0, l1 = prev["lane"][k], st["lane"][k]
            if g["lane_road"][l1] < 0 and l0 in dyn and pred.get(int(l1)) == l0:
                if turn[l1] == 1:
                    assert dirs[l0] == 1
                if turn[l1] == 0:
                    assert dirs[l0] == 0
            if kinds[l1] == 2 and g["lane_road"][l0] >= 0:
                # vehicles already inside a junction lane finish their move
                assert dirs[l1] == 0, "entered a disabled tidal lane"
        prev = st
    assert o.set_lane_direction(0 if kinds[0] == 0 else int(np.where(kinds == 0)[0][0]), 1) == 1
