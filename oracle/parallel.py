"""TEST INFRASTRUCTURE ONLY — the oracle's grid transforms spread over host cores.

``bench.py``'s ``--impl reference`` arm and ``cpu_baseline`` leg time the
reference algorithm on the GPU box's host cores.  The reference itself is
pure Python/numpy that cannot travel to the box, so they run
this module: the same per-order restatement as ``favest_oracle`` (identical
arithmetic — ``forward_order`` / ``adjoint_order``, the ring DFTs of
favest/scalar.py:149,178 and the Clebsch-Gordan stages of
favest/transforms.py:109-146,165-175), with the per-order stage — where the
reference spends >95 % of its time — spread over a pool of
forked worker processes (one per host core, BLAS pinned to one thread each)
instead of one Python thread.  Results are bitwise the serial oracle's.

Never imported by the product package.
"""

from __future__ import annotations

import os

import numpy as np

from . import favest_oracle as O

_STATE: dict = {}


def _init_worker():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl missing
        pass


def _fwd_task(orders):
    st = _STATE
    return [r for m in orders for r in O.forward_order(m, st["spec"], st["w"], st["t"], st["sx"], st["se"], st["lt"])]


def _adj_task(orders):
    st = _STATE
    return [r for m in orders for r in O.adjoint_order(m, st["g"], st["t"], st["sx"], st["se"], st["lt"])]


def _balanced_chunks(lt: int, n_chunks: int, orders=None):
    """Orders (default 0..lt) in chunks of roughly equal work (work of order m
    ~ lt+1-m), heaviest first so the pool's tail is short."""
    orders = range(lt + 1) if orders is None else sorted(set(int(m) for m in orders))
    per = max(1.0, sum(lt + 1 - m for m in orders) / n_chunks)
    chunks, cur, acc = [], [], 0.0
    for m in orders:
        cur.append(m)
        acc += lt + 1 - m
        if acc >= per:
            chunks.append(cur)
            cur, acc = [], 0.0
    if cur:
        chunks.append(cur)
    return chunks


class GridPort:
    """Forward / adjoint FaVeST on one Gauss-Legendre grid with ``procs`` worker
    processes (default: every host core).  Workers are forked per call, so they
    see the current call's arrays without copying them through pipes."""

    def __init__(self, L: int, procs: int | None = None):
        self.L = L
        self.lt = L + 1
        self.th, self.w, self.n_phi = O.gl_grid(L)
        self.t, s = O.ring_cos_sin(self.th)
        self.sx, self.se = O.seed_table(self.lt, s)
        self.procs = max(1, procs or os.cpu_count() or 1)
        self.chunks = _balanced_chunks(self.lt, 8 * self.procs)

    def _run(self, task, orders=None):
        import multiprocessing as mp

        chunks = self.chunks if orders is None else _balanced_chunks(self.lt, 8 * self.procs, orders)
        if self.procs == 1:
            _init_worker()
            return [r for c in chunks for r in task(c)]
        ctx = mp.get_context("fork")
        with ctx.Pool(self.procs, initializer=_init_worker) as pool:
            return [r for part in pool.imap_unordered(task, chunks) for r in part]

    def forward(self, T, orders=None):
        """(N, 3) complex field -> (a, b), favest/transforms.py:79-147.  With
        ``orders`` only the scalar orders those output orders read (|m|-1..|m|+1)
        are computed; the outputs are then meaningful at those orders only."""
        T = np.asarray(T, dtype=np.complex128)
        t1, t2, t3 = T[:, 0], T[:, 1], T[:, 2]
        combos = np.stack([-t1 + 1j * t2, t1 + 1j * t2, t3], axis=1)  # transforms.py:109-112
        n_theta = len(self.th)
        spec = np.fft.fft(combos.reshape(n_theta, self.n_phi, 3), axis=1)  # scalar.py:149
        _STATE.clear()
        _STATE.update(spec=spec, w=self.w, t=self.t, sx=self.sx, se=self.se, lt=self.lt)
        need = None
        if orders is not None:
            need = {x for mo in orders for x in (abs(mo) - 1, abs(mo), abs(mo) + 1) if 0 <= x <= self.lt}
        out = np.zeros((O.flat_size(self.lt), 3), dtype=np.complex128)
        for mm, rows in self._run(_fwd_task, need):
            m = abs(mm)
            ls = np.arange(m, self.lt + 1)
            out[ls * ls + ls + mm] = rows
        _STATE.clear()
        return O.cg_forward_assemble(out, self.L)

    def adjoint(self, a, b, orders=None, spectrum=False):
        """(a, b) -> (N, 3) complex field, favest/transforms.py:150-181; with
        ``spectrum`` the ring spectra (n_theta, n_phi, 3) before the inverse DFT,
        of which only the bins of ``orders`` (default all) are filled."""
        g = O.vsht_adjoint_merged(a, b, self.L)
        _STATE.clear()
        _STATE.update(g=g, t=self.t, sx=self.sx, se=self.se, lt=self.lt)
        n_theta = len(self.th)
        spec = np.zeros((n_theta, self.n_phi, 3), dtype=np.complex128)
        for mm, col in self._run(_adj_task, orders):
            spec[:, mm % self.n_phi, :] = col
        _STATE.clear()
        if spectrum:
            return spec
        out = np.fft.ifft(spec, axis=1) * self.n_phi  # scalar.py:178
        return out.reshape(n_theta * self.n_phi, 3)
