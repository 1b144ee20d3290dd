"""Boundary items of SURVEY §8(b) (VERDICT r01 "Next round" #8): reads into
caller DEVICE buffers (torch tensors) and the caller-provided allocator
(PyTorch's caching allocator backs the handle's device memory)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def simlib():
    import paper_2406_10661_b200 as p
    p.build()
    return p


KEYS = ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v")


@pytest.mark.parametrize("world", [1, 3])
def test_read_state_device_equals_host_read(simlib, world):
    import torch
    scen = synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=1500, seed=21)
    kw = dict(world=world, loopback=True, direct=True) if world > 1 else {}
    g = simlib.Sim.from_scenario(scen, **kw)
    out = None
    for steps in (0, 37, 250):
        g.step(steps)
        out = g.read_state_device(out)              # buffers reused across reads
        torch.cuda.synchronize()
        host = g.read_state()
        for k in KEYS:
            assert np.array_equal(out[k].cpu().numpy(), np.asarray(host[k])), (steps, k)
        assert np.array_equal(out["lane_signal"].cpu().numpy(), host["lane_signal"])
        assert np.array_equal(out["junc_phase"].cpu().numpy()[:g.n_junctions], host["junc_phase"])
        assert out["t"] == host["t"]
    assert (out["status"] == 2).sum().item() > 0 and (out["status"] == 1).sum().item() > 0


def test_torch_caching_allocator_backs_the_handle(simlib):
    import torch
    scen = synth.city(G=8, n_vehicles=6000, seed=25)
    a = simlib.Sim.from_scenario(scen)
    before = torch.cuda.memory_allocated()
    b = simlib.Sim.from_scenario(scen, allocator="torch")
    grew = torch.cuda.memory_allocated() - before
    assert grew >= b.query_sizes()["device_bytes"] > 0
    for sim in (a, b):
        sim.step(120)
    sa, sb = a.read_state(), b.read_state()
    for k in KEYS:
        assert np.array_equal(sa[k], sb[k]), k
    b.destroy()
    assert torch.cuda.memory_allocated() <= before + (1 << 20)
