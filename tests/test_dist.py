"""Multi-process host logic (world_size 2, gloo on CPU): every rank derives the
same batch / order partition, the union covers the work exactly once and the
order blocks are balanced — the contract the NCCL paths rely on."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1908_00041_b200.shard import order_blocks, order_work, rank_env, shard_batch

        r, w, _ = rank_env()
        assert (r, w) == (rank, world)
        B, Lt = 5, 1025
        lo, hi = shard_batch(B, world, rank)
        mine = order_blocks(Lt, world)[rank]
        cover = torch.zeros(B + Lt + 1, dtype=torch.int64)
        cover[lo:hi] += 1
        for m in mine:
            cover[B + m] += 1
        dist.all_reduce(cover)
        work = torch.tensor([sum(order_work(Lt, m) for m in mine)], dtype=torch.int64)
        works = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(works, work)
        if rank == 0:
            q.put((cover.tolist(), [int(x) for x in works]))
    finally:
        dist.destroy_process_group()


def test_partition_over_two_gloo_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    cover, works = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(c == 1 for c in cover)
    assert abs(works[0] - works[1]) <= 1027
