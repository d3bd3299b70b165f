"""Multi-rank host logic on CPU (gloo, world_size 2): batch sharding is a
partition, the final gather returns every rank's rows in order, and the step
time is the max over ranks (bench.py)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_17320_b200.shard import gather_rows, max_over_ranks, shard_range


@pytest.mark.parametrize("n,world", [(8, 1), (8, 2), (7, 2), (3, 8), (0, 4), (16, 8)])
def test_shard_range_partitions(n, world):
    covered = []
    for r in range(world):
        f, c = shard_range(n, world, r)
        covered += list(range(f, f + c))
    assert covered == list(range(n))
    counts = [shard_range(n, world, r)[1] for r in range(world)]
    assert max(counts) - min(counts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, cnt = shard_range(n_total, world, rank)
    # each rank "computes" rows tagged with their global sequence index
    local = torch.arange(first, first + cnt, dtype=torch.float32)[:, None].repeat(1, 3)
    allrows = gather_rows(local)
    t = max_over_ranks(10.0 + rank)
    q.put((rank, allrows[:, 0].tolist(), t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [8, 7])
def test_gather_and_max_over_ranks_gloo(n_total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rows, t in res:
        assert rows == [float(i) for i in range(n_total)]
        assert t == 11.0
