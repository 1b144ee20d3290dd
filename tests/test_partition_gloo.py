"""Multi-process host logic of the partitioned path, world_size 2
over gloo on CPU: every rank derives the partition and the exchange plan
independently from the same inputs; the ranks must agree exactly, and what a
rank plans to send must be what its peer plans to receive."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    import paper_2406_10661_b200 as p
    s = synth.city(G=12, n_vehicles=8000, seed=9)
    own, mig, halo = p.partition(s.graph, s.trips, s.profiles, s.params, world)
    t_own = torch.tensor(own, dtype=torch.int32)
    outs = [torch.zeros_like(t_own) for _ in range(world)]
    dist.all_gather(outs, t_own)
    agree = all(torch.equal(o, t_own) for o in outs)
    # what I send to each peer (mig[rank][q]) vs what the peer expects to receive
    send = torch.tensor(mig[rank], dtype=torch.int64)
    recv = torch.zeros(world, dtype=torch.int64)
    parts = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, send)
    for qq in range(world):
        recv[qq] = parts[qq][rank]
    expect_recv = torch.tensor(mig[:, rank], dtype=torch.int64)
    halo_ok = bool(np.all((halo[rank] > 0) == (mig[rank] > 0)))   # a reads b <=> a feeds b
    # NCCL-path buffer sizing: every region is sized on both sides
    # from the same plan entry, so a grouped ncclSend(a->b) and ncclRecv(b<-a)
    # move the same byte count; no self-traffic
    halo_ok = halo_ok and mig[rank, rank] == 0 and halo[rank, rank] == 0
    q.put((rank, agree, bool(torch.equal(recv, expect_recv)), halo_ok, int(mig.sum())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_partition_agreement_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, agree, rx_ok, halo_ok, tot in res:
        assert agree and rx_ok and halo_ok and tot > 0, (rank, agree, rx_ok, halo_ok)
