"""Order-sharded VSHT across GPUs (the C4 layout).

Each rank owns a contiguous block of rings of the grid (its slice of every
field) and a contiguous range of orders m.  The order ranges balance the
Legendre work actually run per order (``GridPlan.order_cost`` / C ABI
``fv_order_cost``: high orders skip their polar pairs, so their work falls
much faster than Lt+1-m) plus a per-order overhead.  One transpose per
direction:

forward
  1. local ring FFTs of the owned rings (``fv_ring_fft``);
  2. all-to-all: bins ±m of every order owner h needs (its orders plus a
     two-order halo) go to h, so h holds all rings at its orders;
  3. ``fv_forward_orders``: fold + Legendre contraction + CG for h's orders
     and the one-order halo either side that the adjoint's coupling reads.
     a, b come back full-size with those orders filled (m-sharded).

adjoint (input: a, b with the owner's orders ±1 valid — the forward's output,
or full tables)
  1. ``fv_adjoint_orders``: coupling + synthesis of the owned orders into
     compact spectra of every ring;
  2. all-to-all: every ring block goes back to its owner;
  3. local inverse ring FFTs → the owned rings of T.

Both transposes can be cut into ``chunks`` order chunks whose asynchronous
all-to-alls overlap the per-chunk stages.  ``gather_coefficients`` turns
m-sharded a, b into full tables on every rank (entries are disjoint: an
all-reduce of zero-masked tables is exact).

The transport is ``torch.distributed.all_to_all_single`` (NCCL on GPUs, one
process per GPU); ``simulate_forward`` / ``simulate_adjoint`` drive several
ranks' plans in one process with local copies in place of the collective
(used to check the sharded path against the single-plan path on one GPU —
nothing in it waits on another rank's kernels).  The per-rank arithmetic is
the same kernels on the same values as ``GridPlan.forward/adjoint``, so the
sharded results are bitwise identical to the unsharded ones unless a forward
launch with few orders splits its pair chunks over CTAs (then to rounding).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def order_work(Lt: int, m: int) -> int:
    """Legendre work of order m at scalar degree Lt: number of degrees l in [m, Lt]."""
    return max(0, Lt + 1 - m)


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# partition (host logic; gloo-tested)
# ---------------------------------------------------------------------------
def ring_blocks(n_theta: int, world: int) -> list[tuple[int, int]]:
    """Contiguous ring ranges [r0, r1) per rank, sizes differing by at most one."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(n_theta, world)
    out, r = [], 0
    for k in range(world):
        n = base + (1 if k < extra else 0)
        out.append((r, r + n))
        r += n
    return out


def order_weights(Lt: int, cost=None) -> list[float]:
    """Per-order work used to balance the partition: without ``cost``, Lt+1-m degrees
    plus one unit for the order's FFT bins / fold; with ``cost`` (GridPlan.order_cost:
    the (degree, pair) products the contraction of order m really runs -- high orders
    skip their polar pairs, so their work falls faster than Lt+1-m), that plus a
    per-order share for the fold / CG / epilogue of ORDER_OVERHEAD pair-rows."""
    if cost is None:
        return [order_work(Lt, m) + 1 for m in range(Lt + 1)]
    c = [float(x) for x in cost]
    if len(c) != Lt + 1:
        raise ValueError(f"order cost has {len(c)} entries, expected {Lt + 1}")
    over = ORDER_OVERHEAD * sum(c) / max(1, Lt + 1)
    return [x + over for x in c]


#: per-order work that does not shrink with the polar skip (fold, CG, the Legendre
#: kernels' per-order pipeline fill and epilogues), as a fraction of the mean order
#: cost; fitted to the C4 per-rank stage times (tools/c4_rank_share.py)
ORDER_OVERHEAD = 0.08


def order_ranges(Lt: int, world: int, cost=None) -> list[tuple[int, int]]:
    """Contiguous order ranges [m0, m1) over 0..Lt with balanced Legendre work
    (order_weights); the cut points are placed at the cumulative-work quantiles.
    Every rank gets at least one order when world <= Lt+1.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    n = Lt + 1
    if world > n:
        raise ValueError(f"{world} ranks for {n} orders")
    w = order_weights(Lt, cost)
    total = float(sum(w))
    cuts, acc, k = [0], 0.0, 1
    for m in range(n):
        acc += w[m]
        while k < world and acc >= total * k / world:
            cuts.append(m + 1)
            k += 1
    while len(cuts) < world:
        cuts.append(n)
    cuts.append(n)
    # at least one order each (monotone repair from the right)
    for i in range(world - 1, 0, -1):
        cuts[i] = min(cuts[i], cuts[i + 1] - 1)
    for i in range(1, world):
        cuts[i] = max(cuts[i], cuts[i - 1] + 1)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


@dataclass(frozen=True)
class RankLayout:
    """What rank h owns and needs (orders are scalar orders 0..Lt)."""

    rings: tuple[int, int]        # owned rings [r0, r1)
    orders: tuple[int, int]       # owned orders [m0, m1): adjoint synthesis, gathered coefficients
    coef: tuple[int, int]         # forward CG orders [c0, c1): owned ∩ 0..L, plus one halo order each side
    legendre: tuple[int, int]     # forward Legendre orders [l0, l1) feeding coef (one more each side)


def rank_layouts(n_theta: int, L: int, world: int, cost=None) -> list[RankLayout]:
    Lt = L + 1
    rb = ring_blocks(n_theta, world)
    ob = order_ranges(Lt, world, cost)
    out = []
    for h in range(world):
        m0, m1 = ob[h]
        c0, c1 = max(0, m0 - 1), min(L + 1, m1 + 1)  # the synthesis of m0..m1-1 reads orders m0-1..m1
        l0, l1 = max(0, c0 - 1), min(Lt + 1, c1 + 1)  # CG of order c reads F at c-1..c+1 (|-1| = 1)
        out.append(RankLayout(rb[h], (m0, m1), (c0, c1), (l0, l1)))
    return out


def order_chunks(rng: tuple[int, int], Lt: int, chunks: int, cost=None) -> list[tuple[int, int]]:
    """[m0, m1) cut into ``chunks`` contiguous pieces of near-equal Legendre work
    (order_weights; empty pieces when there are fewer orders than chunks)."""
    m0, m1 = rng
    if chunks == 1 or m1 - m0 <= 1:
        return [(m0, m1)] + [(m1, m1)] * (chunks - 1)
    w = order_weights(Lt, cost)[m0:m1]
    total = float(sum(w))
    cuts, acc, k = [m0], 0.0, 1
    for i, m in enumerate(range(m0, m1)):
        acc += w[i]
        while k < chunks and acc >= total * k / chunks:
            cuts.append(m + 1)
            k += 1
    while len(cuts) < chunks:
        cuts.append(m1)
    cuts.append(m1)
    return [(cuts[i], cuts[i + 1]) for i in range(chunks)]


def natural_bins(m0: int, m1: int, n_phi: int):
    """(compact index, natural DFT bin) pairs of orders [m0, m1): +m then −m,
    the −0 duplicate of m = 0 left out."""
    nb = m1 - m0
    pos = [(m - m0, m) for m in range(m0, m1)]
    neg = [(nb + m - m0, (n_phi - m) % n_phi) for m in range(m0, m1) if m != 0]
    return pos + neg


# ---------------------------------------------------------------------------
# kernels (C ABI) — a backend object so that tests can substitute a reference
# ---------------------------------------------------------------------------
class CudaStages:
    """The four sharded building blocks on one GridPlan (``fv_ring_fft``,
    ``fv_forward_orders``, ``fv_adjoint_orders``)."""

    def __init__(self, plan):
        from . import _lib

        self.plan = plan
        self.lib = plan.lib
        self._check = _lib.check

    def _stream(self):
        torch = _torch()
        return torch.cuda.current_stream(self.plan.device).cuda_stream

    # spectra views: (3, B, rings, bins) slices of max-batch buffers, inner dims contiguous
    def fft_fields(self, T_local, S_loc):
        """T_local (B, nloc*n_phi, 3) -> S_loc (3, B, nloc, n_phi) ring spectra."""
        n = self.plan.n_phi
        B, nloc = S_loc.shape[1], S_loc.shape[2]
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            self._check(self.lib.fv_ring_fft(self.plan._h, 0, T_local.data_ptr(), 1, 3 * n, 3, S_loc.data_ptr(),
                                             S_loc.stride(0), n, 1, B * nloc, self._stream()))

    def ifft_fields(self, S_loc, T_local):
        n = self.plan.n_phi
        B, nloc = S_loc.shape[1], S_loc.shape[2]
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            self._check(self.lib.fv_ring_fft(self.plan._h, 1, S_loc.data_ptr(), S_loc.stride(0), n, 1,
                                             T_local.data_ptr(), 1, 3 * n, 3, B * nloc, self._stream()))

    def forward_orders(self, S_own, bin_lo, nb, a, b, legendre, coef):
        """S_own (3, B, n_theta, 2*nb) compact spectra of all rings -> a, b at orders coef."""
        B, nth = S_own.shape[1], S_own.shape[2]
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            self._check(self.lib.fv_forward_orders(
                self.plan._h, S_own.data_ptr(), S_own.stride(0), 2 * nb, 1, bin_lo, nb, a.data_ptr(), b.data_ptr(),
                B, legendre[0], legendre[1], coef[0], coef[1], self._stream()))

    def adjoint_orders(self, a, b, orders, S_own):
        """a, b (orders ±1 valid) -> S_own (3, B, n_theta, 2*nb) compact spectra of orders."""
        B, nth, nb = S_own.shape[1], S_own.shape[2], S_own.shape[3] // 2
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            self._check(self.lib.fv_adjoint_orders(
                self.plan._h, a.data_ptr(), b.data_ptr(), B, orders[0], orders[1], S_own.data_ptr(),
                S_own.stride(0), 2 * nb, 1, orders[0], nb, self._stream()))

    # packed spectra: element (c, ring R, bin j) at rtab[c, R] + j of a flat complex buffer
    # (the per-rank blocks of an all-to-all buffer, read / written in place)
    def forward_orders_packed(self, flat, rtab, B, bin_lo, nb, a, b, legendre, coef):
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            self._check(self.lib.fv_forward_orders_packed(
                self.plan._h, flat.data_ptr(), rtab.data_ptr(), rtab.shape[1], bin_lo, nb, a.data_ptr(), b.data_ptr(),
                B, legendre[0], legendre[1], coef[0], coef[1], self._stream()))

    def adjoint_orders_packed(self, a, b, B, orders, flat, rtab, nb):
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            self._check(self.lib.fv_adjoint_orders_packed(
                self.plan._h, a.data_ptr(), b.data_ptr(), B, orders[0], orders[1], flat.data_ptr(), rtab.data_ptr(),
                rtab.shape[1], orders[0], nb, self._stream()))


# ---------------------------------------------------------------------------
# per-rank plan
# ---------------------------------------------------------------------------
class OrderShardedPlan:
    """Rank ``rank`` of ``world`` in the order-sharded transform of B fields.

    ``stages`` performs the kernels (``CudaStages(GridPlan)`` in production);
    ``n_theta``, ``n_phi``, ``L`` describe the grid; tensors are allocated on
    ``device`` with ``max_batch`` fields.
    """

    def __init__(self, stages, L, n_theta, n_phi, max_batch, rank, world, device, group=None, chunks=1,
                 cost=None):
        torch = _torch()
        if not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} of {world}")
        if chunks < 1:
            raise ValueError("chunks must be >= 1")
        self.stages = stages
        self.L, self.Lt = int(L), int(L) + 1
        self.n_theta, self.n_phi = int(n_theta), int(n_phi)
        self.max_batch = int(max_batch)
        self.rank, self.world = int(rank), int(world)
        self.device = torch.device(device)
        self.group = group
        self.chunks = int(chunks)
        self.cost = None if cost is None else [float(x) for x in cost]
        self.layouts = rank_layouts(self.n_theta, self.L, self.world, self.cost)
        me = self.layouts[self.rank]
        self.me = me
        self.nloc = me.rings[1] - me.rings[0]
        self.K = (self.L + 1) ** 2
        c128 = torch.complex128
        B, n = self.max_batch, self.n_phi
        # local ring spectra: forward FFT output, and the adjoint's inverse-FFT input whose
        # bins no rank owns (n_phi > 2 Lt + 1) must stay zero -- hence two buffers
        self.S_loc = torch.empty((3, B, self.nloc, n), dtype=c128, device=self.device)
        self.S_loc_a = torch.zeros((3, B, self.nloc, n), dtype=c128, device=self.device)
        # per chunk q and rank h: forward coefficient / Legendre order ranges, adjoint orders
        Lt = self.Lt
        self._fc, self._fl, self._ao = [], [], []
        for lay in self.layouts:
            cs = order_chunks(lay.coef, Lt, self.chunks, self.cost)
            self._fc.append(cs)
            self._fl.append([(max(0, c0 - 1), min(Lt + 1, c1 + 1)) if c1 > c0 else (c0, c0) for c0, c1 in cs])
            self._ao.append(order_chunks(lay.orders, Lt, self.chunks, self.cost))
        self._rtabs = {}
        self._send_bins = []  # [q][h]: natural bins of h's chunk-q Legendre orders (+m then -m)
        self._recv_bins = []  # [q][h]: (compact index, natural bin) of h's chunk-q adjoint orders
        for q in range(self.chunks):
            sb, rb = [], []
            for h in range(self.world):
                lo, hi = self._fl[h][q]
                idx = list(range(lo, hi)) + [(n - m) % n for m in range(lo, hi)]
                sb.append(torch.tensor(idx, dtype=torch.long, device=self.device))
                pairs = natural_bins(*self._ao[h][q], n)
                rb.append((torch.tensor([p[0] for p in pairs], dtype=torch.long, device=self.device),
                           torch.tensor([p[1] for p in pairs], dtype=torch.long, device=self.device)))
            self._send_bins.append(sb)
            self._recv_bins.append(rb)

    # ---- packed ring-offset tables -------------------------------------------
    def _rtab(self, B, nb_of, key):
        """(3, B * n_theta) int64 on the device: complex offset of (component c, field b,
        ring r) in a buffer of one block per rank h, block h = [3][B][rings of h][2 nb_of(h)]
        (the all-to-all order).  Cached per key."""
        torch = _torch()
        t = self._rtabs.get(key)
        if t is None:
            n = self.n_theta
            tab = np.zeros((3, B * n), dtype=np.int64)
            off = 0
            for h, lay in enumerate(self.layouts):
                r0, r1 = lay.rings
                nr, w = r1 - r0, 2 * nb_of(h)
                cc, bb, rr = np.meshgrid(np.arange(3), np.arange(B), np.arange(nr), indexing="ij")
                tab[cc, bb * n + r0 + rr] = off + ((cc * B + bb) * nr + rr) * w
                off += 3 * B * nr * w
            t = torch.from_numpy(tab).to(self.device)
            self._rtabs[key] = t
        return t

    # ---- transport -------------------------------------------------------
    def _pack(self, blocks):
        """One flat float64 send buffer of the per-destination complex blocks (each
        written once, by index_select / copy straight into its slice)."""
        torch = _torch()
        sizes = [int(np.prod(shape)) * 2 for shape, _ in blocks]
        flat = torch.empty(sum(sizes), dtype=torch.float64, device=self.device)
        o = 0
        for (shape, fill), k in zip(blocks, sizes):
            fill(torch.view_as_complex(flat[o:o + k].view(-1, 2)).view(shape))
            o += k
        return flat, sizes

    def _all_to_all(self, flat_in, in_splits, out_splits, async_op=False):
        """Returns (work or None, the receive buffer as one flat complex tensor: the
        per-source blocks back to back in rank order)."""
        torch = _torch()
        import torch.distributed as dist

        flat_out = torch.empty(sum(out_splits), dtype=torch.float64, device=self.device)
        work = dist.all_to_all_single(flat_out, flat_in, out_splits, in_splits, group=self.group,
                                      async_op=async_op)
        return work, torch.view_as_complex(flat_out.view(-1, 2))

    # ---- forward ---------------------------------------------------------
    def forward_fft(self, T_local):
        """Local ring FFTs of the owned rings -> S_loc (3, B, nloc, n_phi)."""
        B = int(T_local.shape[0])
        S = self.S_loc[:, :B]
        self.stages.fft_fields(T_local, S)
        return S

    def forward_send(self, S, q=0):
        """Chunk q's per-destination blocks (3, B, nloc, 2 nb_hq): one packed buffer."""
        torch = _torch()
        B = int(S.shape[1])
        blocks = []
        for h in range(self.world):
            idx = self._send_bins[q][h]
            blocks.append(((3, B, self.nloc, int(idx.numel())),
                           lambda out, idx=idx: torch.index_select(S, 3, idx, out=out)))
        return self._pack(blocks)

    def forward_recv_sizes(self, B, q=0):
        lo, hi = self._fl[self.rank][q]
        return [3 * B * (l.rings[1] - l.rings[0]) * 2 * (hi - lo) * 2 for l in self.layouts]

    def forward_finish(self, recv, B, a, b, q=0):
        """Chunk q: fold + Legendre + CG of this rank's chunk-q orders, read in place from
        the receive buffer (one block (3, B, rings of g, 2 nb) per source rank g, in rank
        order) through a ring-offset table: no unpack copy."""
        lo, hi = self._fl[self.rank][q]
        c0, c1 = self._fc[self.rank][q]
        if c1 <= c0:
            return a, b
        nb = hi - lo
        rtab = self._rtab(B, lambda g: nb, ("f", B, q))
        self.stages.forward_orders_packed(recv, rtab, B, lo, nb, a, b, (lo, hi), (c0, c1))
        return a, b

    def forward(self, T_local, a=None, b=None):
        """T_local (B, nloc*n_phi, 3) -> a, b (B, (L+1)^2), valid at this rank's coef orders.

        The transpose runs in ``chunks`` order chunks: every chunk's all-to-all is
        issued asynchronously up front (NCCL's stream carries them back to back), then
        chunk q's Legendre / CG runs as soon as chunk q has arrived, overlapping the
        transfers of the chunks after it."""
        torch = _torch()
        B = int(T_local.shape[0])
        if a is None:
            a = torch.zeros((B, self.K), dtype=torch.complex128, device=self.device)
        if b is None:
            b = torch.zeros((B, self.K), dtype=torch.complex128, device=self.device)
        S = self.forward_fft(T_local)
        pending = []
        for q in range(self.chunks):
            flat, sizes = self.forward_send(S, q)
            work, recvs = self._all_to_all(flat, sizes, self.forward_recv_sizes(B, q), async_op=True)
            pending.append((work, recvs, flat))
        for q, (work, recv, _) in enumerate(pending):
            if work is not None:
                work.wait()
            self.forward_finish(recv, B, a, b, q)
        return a, b

    # ---- adjoint ---------------------------------------------------------
    def adjoint_send(self, a, b, q=0):
        """Chunk q: synthesis of this rank's chunk-q orders written straight into the send
        buffer, one block (3, B, rings of h, 2 nb) per destination rank h (ring-offset
        table: no pack copy).  Returns (flat float64 buffer, per-destination sizes)."""
        torch = _torch()
        B = int(a.shape[0])
        m0, m1 = self._ao[self.rank][q]
        nb = m1 - m0
        sizes = [3 * B * (l.rings[1] - l.rings[0]) * 2 * nb * 2 for l in self.layouts]
        flat = torch.empty(sum(sizes), dtype=torch.float64, device=self.device)
        if nb:
            rtab = self._rtab(B, lambda h: nb, ("a", B, q))
            self.stages.adjoint_orders_packed(a, b, B, (m0, m1), torch.view_as_complex(flat.view(-1, 2)), rtab, nb)
        return flat, sizes

    def adjoint_recv_sizes(self, B, q=0):
        return [3 * B * self.nloc * 2 * (o[q][1] - o[q][0]) * 2 for o in self._ao]

    def adjoint_unpack(self, recv, B, q=0):
        """Chunk q: the received compact bins of every source rank's orders (blocks
        (3, B, nloc, 2 nb_h) in rank order) -> their natural bins of S_loc_a."""
        S = self.S_loc_a[:, :B]
        o = 0
        for h in range(self.world):
            m0, m1 = self._ao[h][q]
            k = 3 * B * self.nloc * 2 * (m1 - m0)
            r = recv[o:o + k]
            o += k
            if m1 <= m0:
                continue
            blk = r.view(3, B, self.nloc, 2 * (m1 - m0))
            ci, nat = self._recv_bins[q][h]
            S.index_copy_(3, nat, blk.index_select(3, ci))

    def adjoint_finish(self, B, T_local):
        self.stages.ifft_fields(self.S_loc_a[:, :B], T_local)
        return T_local

    def adjoint(self, a, b, T_local=None):
        """a, b (B, (L+1)^2) with this rank's orders +-1 valid -> T_local (B, nloc*n_phi, 3).

        Chunk q's synthesis is followed by its asynchronous all-to-all, which then
        overlaps the synthesis of chunk q + 1; the inverse ring FFTs run once every
        chunk has arrived."""
        torch = _torch()
        B = int(a.shape[0])
        if T_local is None:
            T_local = torch.empty((B, self.nloc * self.n_phi, 3), dtype=torch.complex128, device=self.device)
        pending = []
        for q in range(self.chunks):
            flat, sizes = self.adjoint_send(a, b, q)
            work, recvs = self._all_to_all(flat, sizes, self.adjoint_recv_sizes(B, q), async_op=True)
            pending.append((work, recvs, flat))
        for q, (work, recv, _) in enumerate(pending):
            if work is not None:
                work.wait()
            self.adjoint_unpack(recv, B, q)
        return self.adjoint_finish(B, T_local)

    # ---- coefficients ------------------------------------------------------
    def order_mask(self, orders=None):
        """Boolean (K,) mask of the flat entries l*l+l+m with |m| in ``orders`` (default: owned)."""
        torch = _torch()
        m0, m1 = orders or self.me.orders
        k = torch.arange(self.K, device=self.device)
        l = torch.sqrt(k.to(torch.float64)).floor().to(torch.long)
        m = (k - l * l - l).abs()
        return (m >= m0) & (m < m1)

    def gather_coefficients(self, a, b):
        """m-sharded a, b -> full tables on every rank (disjoint entries, exact all-reduce)."""
        torch = _torch()
        import torch.distributed as dist

        mask = self.order_mask()
        out = []
        for x in (a, b):
            y = torch.where(mask, x, torch.zeros((), dtype=x.dtype, device=x.device))
            yr = torch.view_as_real(y).contiguous()
            dist.all_reduce(yr, group=self.group)
            out.append(torch.view_as_complex(yr))
        return out[0], out[1]


def make_plan(L, grid, max_batch, rank, world, device=None, group=None, chunks=1, balance="cost"):
    """Production constructor: one GridPlan on this rank's GPU + its shard layout; the
    transposes run in ``chunks`` order chunks overlapped with the per-order stages
    (default 1: at C4 on 8 ranks a second chunk costs ~0.6 ms of per-chunk launches
    and packing per rank, more than the ~0.4 ms of all-to-all it could hide;
    tools/c4_rank_share.py).
    ``balance="cost"`` partitions the orders by the plan's measured per-order work
    (GridPlan.order_cost, identical on every rank), ``"degrees"`` by Lt+1-m."""
    from .plan import GridPlan

    plan = GridPlan.from_grid(grid, L, max_batch=max_batch, device=device)
    cost = plan.order_cost() if balance == "cost" else None
    return OrderShardedPlan(CudaStages(plan), L, grid.n_theta, grid.n_phi, max_batch, rank, world,
                            plan.device, group, chunks=chunks, cost=cost)


# ---------------------------------------------------------------------------
# in-process simulation of several ranks (checks, one device)
# ---------------------------------------------------------------------------
def simulate_forward(plans, T_locals):
    torch = _torch()
    B = int(T_locals[0].shape[0])
    S = [p.forward_fft(T) for p, T in zip(plans, T_locals)]
    outs = []
    for p in plans:
        a = torch.zeros((B, p.K), dtype=torch.complex128, device=p.device)
        outs.append((a, torch.zeros_like(a)))
    for q in range(plans[0].chunks):
        sends = [_unflatten(p.forward_send(s, q)) for p, s in zip(plans, S)]
        for h, p in enumerate(plans):
            recv = torch.cat([sends[g][h].reshape(-1) for g in range(len(plans))])
            p.forward_finish(recv, B, outs[h][0], outs[h][1], q)
    return outs


def simulate_adjoint(plans, ab):
    torch = _torch()
    B = int(ab[0][0].shape[0])
    for q in range(plans[0].chunks):
        sends = [_unflatten(p.adjoint_send(a, b, q)) for p, (a, b) in zip(plans, ab)]
        for g, p in enumerate(plans):
            p.adjoint_unpack(torch.cat([sends[h][g].reshape(-1) for h in range(len(plans))]), B, q)
    outs = []
    for p in plans:
        T = torch.empty((B, p.nloc * p.n_phi, 3), dtype=torch.complex128, device=p.device)
        outs.append(p.adjoint_finish(B, T))
    return outs


def _unflatten(packed):
    """The per-destination complex blocks of a packed send buffer."""
    torch = _torch()
    flat, sizes = packed
    out, o = [], 0
    for k in sizes:
        out.append(torch.view_as_complex(flat[o:o + k].view(-1, 2)))
        o += k
    return out
