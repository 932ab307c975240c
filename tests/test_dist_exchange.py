"""Host logic of the multi-process executor on CPU: the grouped point-to-
point exchange used for the sparsity-aware row fetch and the feature
all-to-allv, world_size 2 over gloo (127.0.0.1)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_02909_b200.dist_exec import exchange, exchange_counts

    peers = list(range(world))
    # rank r sends r+1 copies of (10r + peer) to every peer, nothing to itself on rank 1
    sends = {p: torch.full((rank + 1,), 10 * rank + p, dtype=torch.int32)
             for p in peers if not (rank == 1 and p == 1)}
    counts = exchange_counts(sends, peers, torch.device("cpu"))
    got = exchange(sends, counts, peers, torch.int32, torch.device("cpu"))
    res = {p: got[p].tolist() for p in got}
    q.put((rank, counts, res))
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, counts, res = q.get(timeout=120)
        out[rank] = (counts, res)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] == {0: 1, 1: 2}
    assert out[0][1][1] == [10, 10] and out[0][1][0] == [0]
    assert out[1][0] == {0: 1, 1: 0}
    assert out[1][1][0] == [1] and out[1][1].get(1, []) == []
