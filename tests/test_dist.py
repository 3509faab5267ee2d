"""Multi-rank host logic on CPU (gloo, world_size 2): sharding of independent samples,
max-over-ranks timing and the gather of per-sample totals."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_03086_b200.dist import gather_totals, max_over_ranks, shard


def test_shard_partitions_units():
    for n in (0, 1, 5, 32, 33):
        for w in (1, 2, 3, 8):
            slices = [shard(n, w, r) for r in range(w)]
            assert slices[0][0] == 0 and slices[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(slices, slices[1:]))
            sizes = [e - b for b, e in slices]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, e = shard(7, world, rank)
        local = torch.arange(b, e, dtype=torch.float64).reshape(-1, 1) * 10.0
        tot = gather_totals(local)
        t = max_over_ranks(1.5 + rank)
        q.put((rank, tot.reshape(-1).tolist(), t))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tot, t in res:
        assert tot == [0.0, 10.0, 20.0, 30.0, 40.0, 50.0, 60.0]
        assert t == 2.5


def test_single_process_identity():
    assert max_over_ranks(3.0) == 3.0
    x = torch.ones(2, 1)
    assert gather_totals(x) is x
