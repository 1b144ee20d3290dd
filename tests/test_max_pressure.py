"""MAX_PRESSURE signal policy (
DESIGN §1.4, readings L38-L41).

Pins of the oracle (CPU):
  * the two-phase worked example of S:336: phase 0 movements 5-0 and 3-1,
    phase 1 movement 2-0 -> pressures 7 vs 2 -> phase 0 (after the yellow);
  * ties -> lowest phase index, and an argmax equal to the running
    phase keeps it (no yellow);
  * brute force: on random grid states, every MAX_PRESSURE junction's next
    state recomputed here from the lane counts and the green table;
  * directional (mirroring Table 2 P:934-935 where MaxPressure's ATT
    is below FixedTime's): on the moderately congested 4x4 grid, MaxPressure's
    ATT <= 0.99 x FixedTime's and its throughput >= 0.99 x, over 3 seeds.
GPU parity: the same pins through the C ABI, and one step from random states
with MAX_PRESSURE junctions bit-identical to the oracle (test_gpu_parity).
"""
import numpy as np
import pytest

import synth

P = 30          # decision period
Y = 3           # yellow steps (L21)


def _decide(sim_cls, make, counts, phase, **kw):
    """Junction state after one step from (phase, elapsed = P - 1) with the
    given initial lane counts (A, B, C, D, E, F)."""
    sc, _ = synth.pressure_junction(counts, period=P)
    sim = make(sc, **kw)
    st = sim.read_state()
    st["junc_phase"][:] = phase
    st["junc_pending"][:] = phase
    st["junc_elapsed"][:] = P - 1
    st["junc_yellow_left"][:] = 0
    sim.load_state(st)
    sim.step(1)
    return sim, sim.read_state()


def _oracle(oracle_lib):
    def make(sc, **kw):
        return oracle_lib.Oracle(sc)
    return make


def test_worked_example_S336(oracle_lib):
    sim, st = _decide(None, _oracle(oracle_lib), [5, 3, 2, 0, 1, 0], phase=1)
    # pressure(phase 0) = (5-0) + (3-1) = 7 > pressure(phase 1) = 2 - 0 = 2
    assert st["junc_phase"][0] == 1 and st["junc_yellow_left"][0] == Y
    assert st["junc_pending"][0] == 0
    sim.step(Y)
    st = sim.read_state()
    assert st["junc_phase"][0] == 0 and st["junc_yellow_left"][0] == 0
    assert st["junc_elapsed"][0] == 0


def test_tie_lowest_index_and_keep(oracle_lib):
    # tie 6 = (4-0) + (3-1) vs 6 - 0: lowest index (phase 0) wins -> switch from 1
    _, st = _decide(None, _oracle(oracle_lib), [4, 3, 6, 0, 1, 0], phase=1)
    assert st["junc_yellow_left"][0] == Y and st["junc_pending"][0] == 0
    # phase 1 strictly larger while running phase 1: kept, elapsed restarts
    _, st = _decide(None, _oracle(oracle_lib), [1, 1, 6, 0, 1, 0], phase=1)
    assert st["junc_phase"][0] == 1 and st["junc_yellow_left"][0] == 0
    assert st["junc_elapsed"][0] == 0
    # below the period nothing is decided
    sc, _ = synth.pressure_junction([5, 3, 2, 0, 1, 0], period=P)
    o = oracle_lib.Oracle(sc)
    o.step(1)
    st = o.read_state()
    assert st["junc_phase"][0] == 0 and st["junc_elapsed"][0] == 1


def _brute_next(g, st, j, period):
    """Next (phase, elapsed, yellow, pending) of MAX_PRESSURE junction j from
    state st (no request pending), written from L38-L41 directly."""
    cnt = np.bincount(st["lane"][st["status"] == 1], minlength=len(g["lane_length"]))
    lanes = g["junc_lanes"][g["junc_lane_offsets"][j]:g["junc_lane_offsets"][j + 1]]
    ns = len(lanes)
    K = g["junc_phase_offsets"][j + 1] - g["junc_phase_offsets"][j]
    # green rows: junctions before j contribute ns_i * K_i bytes each
    off = sum(int(np.diff(g["junc_lane_offsets"])[i] * np.diff(g["junc_phase_offsets"])[i])
              for i in range(j))
    green = g["phase_green"][off:off + ns * K].reshape(K, ns)
    pred = {int(s): int(l) for l in range(len(g["lane_length"]))
            for s in g["succ_lanes"][g["succ_offsets"][l]:g["succ_offsets"][l + 1]]}
    succ = {int(l): int(g["succ_lanes"][g["succ_offsets"][l]]) for l in lanes}
    press = [sum(int(cnt[pred[int(l)]]) - int(cnt[succ[int(l)]])
                 for q, l in enumerate(lanes) if green[k, q]) for k in range(K)]
    ph, el, y, pe = (int(st["junc_phase"][j]), int(st["junc_elapsed"][j]),
                     int(st["junc_yellow_left"][j]), int(st["junc_pending"][j]))
    if y > 0:
        y -= 1
        if y == 0:
            ph, el = pe, 0
        return ph, el, y, pe
    el += 1
    if el >= period:
        best = int(np.argmax(press))          # first maximum = lowest index
        if best == ph:
            el = 0
        else:
            y, pe = Y, best
    return ph, el, y, pe


def test_brute_force_random_states(oracle_lib):
    sc = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=61,
                    policy=synth.POLICY_MAXP)
    g = sc.graph
    o = oracle_lib.Oracle(sc)
    checked = 0
    for seed in range(6):
        st = synth.random_state(sc, seed=300 + seed)
        o.load_state({k: (v.astype(np.float64) if k in ("s", "v") else v) for k, v in st.items()})
        before = o.read_state()
        o.step(1)
        after = o.read_state()
        for j in np.where(before["junc_policy"] == synth.POLICY_MAXP)[0]:
            exp = _brute_next(g, before, int(j), P)
            got = (after["junc_phase"][j], after["junc_elapsed"][j],
                   after["junc_yellow_left"][j], after["junc_pending"][j])
            assert tuple(int(x) for x in got) == exp, (seed, j, got, exp)
            checked += 1
    assert checked > 20


def test_directional_maxpressure_vs_fixedtime(oracle_lib):
    for seed in (2, 3, 4):
        res = {}
        for pol in (synth.POLICY_FIXED, synth.POLICY_MAXP):
            sc = synth.grid(seed=seed, n_trips=2500, policy=pol)
            o = oracle_lib.Oracle(sc)
            o.step(3600)
            m = o.metrics()
            res[pol] = (m["n_finished"], m["sum_travel_steps"] / m["n_finished"])
        (tp_f, att_f), (tp_m, att_m) = res[synth.POLICY_FIXED], res[synth.POLICY_MAXP]
        assert att_m <= 0.99 * att_f, (seed, res)
        assert tp_m >= 0.99 * tp_f, (seed, res)


@pytest.mark.gpu
def test_worked_example_gpu():
    import paper_2406_10661_b200 as p
    p.build()
    make = lambda sc, **kw: p.Sim.from_scenario(sc)
    sim, st = _decide(None, make, [5, 3, 2, 0, 1, 0], phase=1)
    assert st["junc_phase"][0] == 1 and st["junc_yellow_left"][0] == Y
    assert st["junc_pending"][0] == 0
    sim.step(Y)
    st = sim.read_state()
    assert st["junc_phase"][0] == 0 and st["junc_elapsed"][0] == 0
    _, st = _decide(None, make, [4, 3, 6, 0, 1, 0], phase=1)
    assert st["junc_yellow_left"][0] == Y and st["junc_pending"][0] == 0
    _, st = _decide(None, make, [1, 1, 6, 0, 1, 0], phase=1)
    assert st["junc_phase"][0] == 1 and st["junc_elapsed"][0] == 0
