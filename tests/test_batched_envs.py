"""Batched environments (the RL workload of P:146,
P:817-818): independent networks stepped by one call, as one graph with
disconnected components (synth.batch).  With the per-vehicle Philox key /
counter id of sim_params, every environment must behave exactly like its
standalone run:
  * exact mode: each environment bit-identical to the oracle run of that
    environment alone (store_fp32), state and per-group metrics;
  * default fp32 path: each environment bit-identical to the GPU run of that
    environment alone (nothing couples environments; per-vehicle arithmetic
    depends only on the vehicle's own snapshot neighbourhood).
"""
import numpy as np
import pytest

import synth

KEYS_INT = ("status", "cursor", "wait_steps", "insert_time", "arrive_time")
MKEYS = ("n_pending", "n_driving", "n_finished", "vehicle_steps", "sum_travel_steps",
         "sum_wait_steps_finished", "sum_depart_delay", "n_lane_changes", "n_handoffs",
         "n_inserted")


def _envs():
    return [synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=800, seed=71),
            synth.grid(rows=2, cols=3, road_len=250.0, lanes=3, n_trips=600, seed=72,
                       tidal=True, dynamic=True),
            synth.grid(rows=3, cols=2, road_len=200.0, lanes=2, n_trips=700, seed=73,
                       policy=synth.POLICY_MAXP)]


def _slices(B):
    vo = np.concatenate([[0], np.cumsum(B.meta["env_trips"])])
    lo = np.concatenate([[0], np.cumsum(B.meta["env_lanes"])])
    jo = np.concatenate([[0], np.cumsum(B.meta["env_junctions"])])
    return vo, lo, jo


def _env_state(st, e, vo, lo, jo):
    sl = slice(vo[e], vo[e + 1])
    out = {k: np.asarray(st[k])[sl] for k in KEYS_INT + ("s", "v")}
    lane = np.asarray(st["lane"])[sl].copy()
    lane[lane >= 0] -= lo[e]
    out["lane"] = lane
    for k in ("junc_phase", "junc_elapsed", "junc_yellow_left", "junc_pending", "junc_policy"):
        out[k] = np.asarray(st[k])[jo[e]:jo[e + 1]]
    return out


def test_batch_input_is_a_disjoint_union():
    envs = _envs()
    B = synth.batch(envs)
    vo, lo, jo = _slices(B)
    g = B.graph
    assert len(g["lane_length"]) == lo[-1] and B.n_trips == vo[-1]
    for e, sc in enumerate(envs):
        # every successor of an environment's lane stays in that environment
        for l in range(lo[e], lo[e + 1]):
            succ = g["succ_lanes"][g["succ_offsets"][l]:g["succ_offsets"][l + 1]]
            assert np.all((succ >= lo[e]) & (succ < lo[e + 1]))
        assert np.array_equal(B.trips["start_lane"][vo[e]:vo[e + 1]] - lo[e], sc.trips["start_lane"])
    assert np.array_equal(B.params["vehicle_rng_id"][vo[1]:vo[2]], np.arange(envs[1].n_trips))


@pytest.mark.gpu
def test_batched_exact_equals_standalone_oracle(oracle_lib):
    import paper_2406_10661_b200 as p
    p.build()
    envs = _envs()
    B = synth.batch(envs)
    vo, lo, jo = _slices(B)
    g = p.Sim.from_scenario(B, exact_mode=True)
    orcs = [oracle_lib.Oracle(sc, store_fp32=True) for sc in envs]
    for chunk in range(3):
        g.step(100)
        for o in orcs:
            o.step(100)
        gs = g.read_state()
        gm = g.read_group_metrics(len(envs))
        for e, o in enumerate(orcs):
            es, os_ = _env_state(gs, e, vo, lo, jo), o.read_state()
            for k in KEYS_INT + ("lane", "junc_phase", "junc_elapsed", "junc_yellow_left"):
                assert np.array_equal(es[k], os_[k]), (chunk, e, k)
            d = os_["status"] == 1
            assert np.array_equal(es["s"][d].astype(np.float64), os_["s"][d]), (chunk, e)
            om = o.metrics()
            for k in MKEYS:
                assert gm[e][k] == om[k], (chunk, e, k, gm[e][k], om[k])


@pytest.mark.gpu
def test_batched_fp32_equals_standalone_gpu():
    import paper_2406_10661_b200 as p
    p.build()
    envs = _envs()
    B = synth.batch(envs)
    vo, lo, jo = _slices(B)
    g = p.Sim.from_scenario(B)
    solo = [p.Sim.from_scenario(sc) for sc in envs]
    g.step(300)
    for s in solo:
        s.step(300)
    gs = g.read_state()
    gm = g.read_group_metrics(len(envs))
    for e, s in enumerate(solo):
        es, ss = _env_state(gs, e, vo, lo, jo), s.read_state()
        for k in KEYS_INT + ("lane", "s", "v", "junc_phase"):
            assert np.array_equal(es[k], ss[k]), (e, k)
        sm = s.read_metrics()
        for k in MKEYS + ("n_guard_hits",):
            assert gm[e][k] == sm[k], (e, k)
