"""Direct peer-memory transport across processes (SURVEY §8(f) NEXT-2,
DESIGN §6.1), exercised for real on one GPU: two processes, one partition
each, buffers mapped with CUDA IPC, handles all-gathered over a gloo process
group, a device barrier per step.  The union of the two ranks' states and the
rank-summed metrics must equal the single-partition run bit for bit (P-PART).
On a multi-GPU box the same code maps NVLink peer memory."""
import os
import socket
import tempfile

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

STEPS = 80


def _scen(name):
    if name == "city":
        return synth.city(G=12, n_vehicles=20000, seed=13)
    return synth.grid(rows=4, cols=4, road_len=250.0, lanes=2, n_trips=3000, seed=12,
                      depart_window=400, policy=synth.POLICY_MAXP)


def _worker(rank, world, port, name, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2406_10661_b200 as p
    scen = _scen(name)
    g = p.Sim.from_scenario(scen, world=world, rank=rank, direct=True, device=0)
    g.connect_process_group()
    g.step(STEPS // 2)
    moved = g.repartition()                          # NEXT-2 rebalance by current load
    g.step(STEPS - STEPS // 2)
    st = g.read_state()
    sg = g.read_state(global_view=True)                   # every rank's vehicles via peer memory
    m = g.read_metrics(lane_stats=True)
    np.savez(os.path.join(out_dir, f"g{rank}.npz"), **{k: np.asarray(v) for k, v in sg.items()})
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), moved=moved,
             **{k: np.asarray(v) for k, v in st.items()},
             **{"m_" + k: np.asarray(v) for k, v in m.items() if v is not None})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world", [("city", 2), ("grid_maxpressure", 2), ("city", 3)])
def test_multi_process_direct_transport(name, world):
    import torch.multiprocessing as mp
    import paper_2406_10661_b200 as p
    p.build()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), name, d), nprocs=world,
                           join=True, start_method="spawn")
        rs = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]
        gs = [dict(np.load(os.path.join(d, f"g{r}.npz"))) for r in range(world)]
    ref = p.Sim.from_scenario(_scen(name))
    ref.step(STEPS)
    s1 = ref.read_state()
    m1 = ref.read_metrics(lane_stats=True)
    assert len({int(r["moved"]) for r in rs}) == 1 and int(rs[0]["moved"]) > 0
    # union of the partitions: each DRIVING vehicle is reported by its owner only
    drv = np.stack([r["status"] == 1 for r in rs])
    assert (drv.sum(0) <= 1).all()
    assert np.array_equal(drv.any(0), s1["status"] == 1)
    fin = np.stack([r["status"] == 2 for r in rs]).any(0)
    assert np.array_equal(fin, s1["status"] == 2)
    for k in ("lane", "cursor", "wait_steps", "s", "v"):
        u = np.zeros_like(s1[k])
        for q, r in enumerate(rs):
            u[drv[q]] = r[k][drv[q]]
        m = s1["status"] == 1
        assert np.array_equal(u[m], s1[k][m]), k
    for k in ("n_pending", "n_driving", "n_finished", "vehicle_steps", "sum_travel_steps",
              "n_lane_changes", "n_handoffs", "n_inserted"):
        for r in rs:                                 # every rank sees the global totals
            assert int(r["m_" + k]) == m1[k], (k, int(r["m_" + k]), m1[k])
    for r in rs:
        assert np.array_equal(r["m_lane_count"], m1["lane_count"])
    for k in ("junc_phase", "lane_signal"):
        for r in rs:
            assert np.array_equal(r[k], s1[k]), k
    assert m1["n_handoffs"] > 0
    for gq in gs:                                    # the global view on every rank = one partition
        for k in ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v"):
            assert np.array_equal(gq[k], s1[k]), k


def _stall_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2406_10661_b200 as p
    scen = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=500, seed=5)
    g = p.Sim.from_scenario(scen, world=world, rank=rank, direct=True, device=0, barrier_timeout_ms=2000)
    g.connect_process_group()
    result = "none"
    if rank == 0:                                    # rank 1 never steps
        g.step(1)
        try:
            g.sync()
            result = "no error"
        except p.SimError as e:
            result = f"{e.status}:{e}"
        try:
            g.step(1)                                # the handle stays sticky
            result += "|stepped"
        except p.SimError as e:
            result += f"|{e.status}"
        with open(os.path.join(out_dir, "r0.txt"), "w") as f:
            f.write(result)
    dist.barrier()                                   # rank 1 keeps its buffers mapped until here
    dist.destroy_process_group()


def test_peer_that_stops_stepping_does_not_hang():
    """A rank whose peer never reaches the barrier gets a sticky SIM_E_STATE
    after the barrier timeout instead of a hung GPU."""
    import torch.multiprocessing as mp
    import paper_2406_10661_b200 as p
    p.build()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_stall_worker, args=(2, _free_port(), d), nprocs=2, join=True,
                           start_method="spawn")
        res = open(os.path.join(d, "r0.txt")).read()
    assert res.startswith("6:") and "barrier timed out" in res, res
    assert res.endswith("|6"), res


def _route_worker(rank, world, port, out_dir):
    import json as _json
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2406_10661_b200 as p
    scen = _scen("grid_maxpressure")
    req = _json.load(open(os.path.join(out_dir, "req.json")))
    g = p.Sim.from_scenario(scen, world=world, rank=rank, direct=True, device=0)
    g.connect_process_group()
    g.step(40)
    g.set_vehicle_route_batch(req["vids"], req["routes"], req["end_s"])   # SPMD, same batch
    g.step(40)
    st = g.read_state()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **{k: np.asarray(v) for k, v in st.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_multi_process_set_vehicle_route():
    """NEXT-4's set_vehicle_route across processes: a vehicle is located by
    the rank that owns it (sum of the ranks' answers), so every rank validates
    and applies the batch identically; the result equals one partition."""
    import json as _json
    import torch.multiprocessing as mp
    import paper_2406_10661_b200 as p
    from test_controllables import _reroutes
    p.build()
    scen = _scen("grid_maxpressure")
    ref = p.Sim.from_scenario(scen)
    ref.step(40)
    req = _reroutes(scen, ref.read_state(), np.random.default_rng(3))
    assert any(True for _ in req)
    vids, routes, ends = [k for k, _, _ in req], [r for _, r, _ in req], [e for _, _, e in req]
    ref.set_vehicle_route_batch(vids, routes, ends)
    ref.step(40)
    s1 = ref.read_state()
    world = 2
    with tempfile.TemporaryDirectory() as d:
        _json.dump({"vids": vids, "routes": [list(map(int, r)) for r in routes], "end_s": ends},
                   open(os.path.join(d, "req.json"), "w"))
        mp.start_processes(_route_worker, args=(world, _free_port(), d), nprocs=world,
                           join=True, start_method="spawn")
        rs = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]
    drv = np.stack([r["status"] == 1 for r in rs])
    assert np.array_equal(drv.any(0), s1["status"] == 1)
    for k in ("lane", "cursor", "s", "v"):
        u = np.zeros_like(s1[k])
        for q, r in enumerate(rs):
            u[drv[q]] = r[k][drv[q]]
        m = s1["status"] == 1
        assert np.array_equal(u[m], s1[k][m]), k
