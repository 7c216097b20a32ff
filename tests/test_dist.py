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
        from paper_1908_00041_b200.dist import order_work, rank_layouts

        n_theta, L = 1026, 1024
        Lt = L + 1
        me = rank_layouts(n_theta, L, world)[rank]
        cover = torch.zeros(n_theta + Lt + 1, dtype=torch.int64)
        cover[me.rings[0]:me.rings[1]] += 1
        cover[n_theta + me.orders[0]:n_theta + me.orders[1]] += 1
        dist.all_reduce(cover)
        work = torch.tensor([sum(order_work(Lt, m) + 1 for m in range(*me.orders))], dtype=torch.int64)
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
    assert all(c == 1 for c in cover)  # every ring and every order owned exactly once
    assert abs(works[0] - works[1]) <= 2 * 1027


# ---------------------------------------------------------------------------
# order-sharded transform (paper_1908_00041_b200/dist.py) over gloo, oracle stages
# ---------------------------------------------------------------------------
def _field_and_coeffs(L, B, seed):
    import numpy as np

    import oracle as O

    th, w, n = O.gl_grid(L)
    rng = np.random.default_rng(seed)
    ab = [O.coef(rng, L, "inv") for _ in range(B)]
    A = np.stack([x[0] for x in ab])
    Bc = np.stack([x[1] for x in ab])
    T = np.stack([O.vsht_adjoint_grid(A[f], Bc[f], L, th, n) for f in range(B)])
    T = T + np.stack([O.tangent_noise(rng, O.grid_points(th, n), 0.05) for _ in range(B)])
    return th, w, n, T


def _sharded_worker(rank, world, port, q, chunks=1):
    import numpy as np

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from dist_oracle_stages import OracleStages
        from paper_1908_00041_b200.dist import OrderShardedPlan

        L, B = 9, 2
        th, w, n, T = _field_and_coeffs(L, B, 11)
        nth = len(th)
        plan = OrderShardedPlan(OracleStages(L, th, w, n), L, nth, n, B, rank, world, "cpu", chunks=chunks)
        r0, r1 = plan.me.rings
        T_local = torch.from_numpy(T.reshape(B, nth, n, 3)[:, r0:r1].reshape(B, -1, 3).copy())
        a, b = plan.forward(T_local)
        ag, bg = plan.gather_coefficients(a, b)
        Tl = plan.adjoint(a, b)  # m-sharded input: the owner's orders +-1 are valid
        mx = max(l.rings[1] - l.rings[0] for l in plan.layouts) * n  # gloo all_gather wants equal sizes
        pad = torch.zeros((B, mx, 3), dtype=torch.complex128)
        pad[:, :Tl.shape[1]] = Tl
        parts = [torch.zeros_like(pad) for _ in plan.layouts]
        dist.all_gather(parts, pad)
        parts = [p[:, :(l.rings[1] - l.rings[0]) * n] for p, l in zip(parts, plan.layouts)]
        if rank == 0:
            ra = np.stack([O.vsht_forward_grid(T[f], th, w, n, L)[0] for f in range(B)])
            rb = np.stack([O.vsht_forward_grid(T[f], th, w, n, L)[1] for f in range(B)])
            ef = O.rel_l2(np.concatenate([ag.numpy(), bg.numpy()], 1), np.concatenate([ra, rb], 1))
            Tfull = torch.cat([p.view(B, -1, n, 3) for p in parts], 1).reshape(B, -1, 3).numpy()
            Tref = np.stack([O.vsht_adjoint_grid(ra[f], rb[f], L, th, n) for f in range(B)])
            q.put((ef, O.rel_l2(Tfull, Tref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 3])
def test_order_sharded_transform_over_two_gloo_ranks(chunks):
    """world 2 over gloo; chunks 3: the transposes split into order chunks whose
    asynchronous all-to-alls overlap the per-chunk stages (dist.py forward / adjoint)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q, chunks)) for r in range(world)]
    for p in procs:
        p.start()
    ef, ea = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ef <= 1e-13 and ea <= 1e-13


@pytest.mark.parametrize("world,chunks", [(1, 1), (3, 1), (4, 1), (1, 3), (3, 2), (4, 5)])
def test_order_sharded_simulated_ranks_match_oracle(world, chunks):
    """The same driver, ranks simulated in one process (local copies for the transposes)."""
    import numpy as np

    import oracle as O
    from dist_oracle_stages import OracleStages
    from paper_1908_00041_b200.dist import OrderShardedPlan, simulate_adjoint, simulate_forward

    L, B = 8, 2
    th, w, n, T = _field_and_coeffs(L, B, 5 + world)
    nth = len(th)
    plans = [OrderShardedPlan(OracleStages(L, th, w, n), L, nth, n, 3, r, world, "cpu", chunks=chunks)
             for r in range(world)]
    T4 = T.reshape(B, nth, n, 3)
    Tl = [torch.from_numpy(T4[:, p.me.rings[0]:p.me.rings[1]].reshape(B, -1, 3).copy()) for p in plans]
    outs = simulate_forward(plans, Tl)
    ls, ms = O.degrees_orders(L)
    ref = [O.vsht_forward_grid(T[f], th, w, n, L) for f in range(B)]
    for p, (a, b) in zip(plans, outs):
        sel = torch.from_numpy((np.abs(ms) >= p.me.coef[0]) & (np.abs(ms) < p.me.coef[1]))
        for f in range(B):
            assert O.rel_l2(a[f][sel].numpy(), ref[f][0][sel.numpy()]) <= 1e-13
            assert O.rel_l2(b[f][sel].numpy(), ref[f][1][sel.numpy()]) <= 1e-13
    Tout = simulate_adjoint(plans, outs)
    Tfull = torch.cat([t.view(B, -1, n, 3) for t in Tout], 1).reshape(B, -1, 3).numpy()
    for f in range(B):
        Tref = O.vsht_adjoint_grid(ref[f][0], ref[f][1], L, th, n)
        assert O.rel_l2(Tfull[f], Tref) <= 1e-13


def test_order_partition_properties():
    from paper_1908_00041_b200.dist import natural_bins, order_ranges, order_work, rank_layouts, ring_blocks

    for Lt, world in ((1025, 8), (4097, 8), (33, 4), (10, 11), (5, 2)):
        rr = order_ranges(Lt, world)
        assert rr[0][0] == 0 and rr[-1][1] == Lt + 1
        assert all(a < b for a, b in rr) and all(rr[i][1] == rr[i + 1][0] for i in range(world - 1))
        if world <= 8 and Lt > 100:
            works = [sum(order_work(Lt, m) + 1 for m in range(a, b)) for a, b in rr]
            assert max(works) - min(works) <= 2 * (Lt + 2)
    assert ring_blocks(10, 3) == [(0, 4), (4, 7), (7, 10)]
    for lay in rank_layouts(1026, 1024, 8):
        m0, m1 = lay.orders
        assert lay.coef[0] <= max(0, m0 - 1) and lay.coef[1] >= min(1025, m1 + 1)
        assert lay.legendre[0] <= max(0, lay.coef[0] - 1) and lay.legendre[1] >= min(1026, lay.coef[1] + 1)
    nb = natural_bins(0, 3, 20)
    assert nb == [(0, 0), (1, 1), (2, 2), (4, 19), (5, 18)]


def test_order_chunks_cover_and_balance():
    from paper_1908_00041_b200.dist import order_chunks, order_work

    for rng, Lt, k in (((0, 1026), 1025, 4), ((300, 700), 1025, 3), ((5, 7), 1025, 4), ((0, 4098), 4097, 8),
                       ((9, 10), 9, 2)):
        cs = order_chunks(rng, Lt, k)
        assert len(cs) == k and cs[0][0] == rng[0] and cs[-1][1] == rng[1]
        assert all(cs[i][1] == cs[i + 1][0] for i in range(k - 1)) and all(a <= b for a, b in cs)
        if rng[1] - rng[0] >= 100:
            works = [sum(order_work(Lt, m) + 1 for m in range(a, b)) for a, b in cs]
            assert max(works) - min(works) <= 2 * (Lt + 2)
