"""Device plans: the batched torch API over the C ABI.

``GridPlan`` owns one ``fvPlan`` for a tensor grid (ring tables, Legendre
seeds, recurrence coefficients, cuFFT plans and workspaces) and runs the
forward / adjoint VSHT on ``(B, N, 3)`` / ``(B, K)`` complex128 CUDA tensors.
``PointsPlan`` does the same at scattered points: the adjoint, and the
forward on weighted rules without tensor-grid structure (the direct route).

All tensors stay on the device; calls are asynchronous on the current torch
stream (``torch.cuda.current_stream``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _torch():
    import torch

    return torch


def _stream_ptr(device) -> ctypes.c_void_p:
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev(device):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("favest_b200 needs a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def _check_tensor(x, shape, name, device):
    torch = _torch()
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if x.dtype != torch.complex128:
        raise ValueError(f"{name} must be complex128, got {x.dtype}")
    if tuple(x.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(x.shape)}, expected {tuple(shape)}")
    if x.device != device:
        raise ValueError(f"{name} is on {x.device}, plan is on {device}")
    return x.contiguous()


class GridPlan:
    """Forward / adjoint VSHT of vector degree ``lmax`` on one tensor grid."""

    def __init__(self, lmax, ring_thetas, ring_weights, n_phi, max_batch=1, device=None):
        self.lib = _lib.load()
        self.device = _dev(device)
        self.lmax = int(lmax)
        th = np.ascontiguousarray(ring_thetas, dtype=np.float64)
        w = np.ascontiguousarray(ring_weights, dtype=np.float64)
        if th.shape != w.shape or th.ndim != 1:
            raise ValueError("ring_thetas and ring_weights must be matching 1-d arrays")
        self.n_theta = int(th.size)
        self.n_phi = int(n_phi)
        self.max_batch = int(max_batch)
        self.n_points = self.n_theta * self.n_phi
        self.n_coeffs = (self.lmax + 1) ** 2
        handle = ctypes.c_void_p()
        dp = ctypes.POINTER(ctypes.c_double)
        with _torch().cuda.device(self.device):
            _lib.check(self.lib.fv_plan_create_grid(
                ctypes.byref(handle), self.lmax, self.n_theta, self.n_phi,
                th.ctypes.data_as(dp), w.ctypes.data_as(dp), self.max_batch, self.device.index))
        self._h = handle
        info = [ctypes.c_int() for _ in range(5)]
        _lib.check(self.lib.fv_plan_info(self._h, *[ctypes.byref(x) for x in info]))
        self.n_pairs = info[3].value
        self.folded = bool(info[4].value)

    @classmethod
    def from_grid(cls, grid, lmax, max_batch=1, device=None):
        return cls(lmax, grid.ring_thetas, grid.ring_weights, grid.n_phi, max_batch, device)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.fv_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def order_cost(self) -> np.ndarray:
        """(lmax+2,) float64: the (degree, ring pair) products the contraction of each
        order m runs (pairs counted from their polar start); fv_order_cost."""
        out = np.zeros(self.lmax + 2, dtype=np.float64)
        _lib.check(self.lib.fv_order_cost(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def set_profiling(self, enable: bool = True):
        _lib.check(self.lib.fv_set_profiling(self._h, int(bool(enable))))

    STAGES = ("fft", "fold", "legendre", "cg")

    def stage_ms(self) -> dict:
        """Accumulated stage times (ms) since set_profiling(True)."""
        return {n: self.lib.fv_stage_ms(self._h, i) for i, n in enumerate(self.STAGES)}

    def stage_counts(self) -> dict:
        return {n: self.lib.fv_stage_count(self._h, i) for i, n in enumerate(self.STAGES)}

    def forward(self, T, a=None, b=None):
        """T (B, N, 3) complex128 -> (a, b), each (B, (lmax+1)**2) complex128."""
        torch = _torch()
        B = int(T.shape[0]) if T.dim() == 3 else -1
        T = _check_tensor(T, (B, self.n_points, 3), "T", self.device)
        if a is None:
            a = torch.empty((B, self.n_coeffs), dtype=torch.complex128, device=self.device)
        if b is None:
            b = torch.empty((B, self.n_coeffs), dtype=torch.complex128, device=self.device)
        a = _check_tensor(a, (B, self.n_coeffs), "a", self.device)
        b = _check_tensor(b, (B, self.n_coeffs), "b", self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_forward_grid(
                self._h, T.data_ptr(), a.data_ptr(), b.data_ptr(), B, _stream_ptr(self.device)))
        return a, b

    def adjoint(self, a, b, T=None):
        """(a, b) (B, (lmax+1)**2) complex128 -> T (B, N, 3) complex128."""
        torch = _torch()
        B = int(a.shape[0]) if a.dim() == 2 else -1
        a = _check_tensor(a, (B, self.n_coeffs), "a", self.device)
        b = _check_tensor(b, (B, self.n_coeffs), "b", self.device)
        if T is None:
            T = torch.empty((B, self.n_points, 3), dtype=torch.complex128, device=self.device)
        T = _check_tensor(T, (B, self.n_points, 3), "T", self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_adjoint_grid(
                self._h, a.data_ptr(), b.data_ptr(), T.data_ptr(), B, _stream_ptr(self.device)))
        return T

    # scalar transforms of degree lmax <= self.lmax + 1 (favest/scalar.py:146-184)
    def forward_scalar(self, f, lmax):
        """f (B, N) complex128 -> (B, (lmax+1)**2) complex128 (forward_sht_fast)."""
        torch = _torch()
        B = int(f.shape[0]) if f.dim() == 2 else -1
        f = _check_tensor(f, (B, self.n_points), "f", self.device)
        out = torch.empty((B, (lmax + 1) ** 2), dtype=torch.complex128, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_forward_scalar_grid(
                self._h, f.data_ptr(), out.data_ptr(), int(lmax), B, _stream_ptr(self.device)))
        return out

    def adjoint_scalar(self, g, lmax):
        """g (B, (lmax+1)**2) complex128 -> f (B, N) complex128 (adjoint_sht_fast)."""
        torch = _torch()
        B = int(g.shape[0]) if g.dim() == 2 else -1
        g = _check_tensor(g, (B, (lmax + 1) ** 2), "g", self.device)
        f = torch.empty((B, self.n_points), dtype=torch.complex128, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_adjoint_scalar_grid(
                self._h, g.data_ptr(), f.data_ptr(), int(lmax), B, _stream_ptr(self.device)))
        return f


class PointsPlan:
    """Adjoint and forward (direct-route) VSHT of vector degree ``lmax`` at
    scattered unit points."""

    def __init__(self, lmax, max_batch=1, device=None):
        self.lib = _lib.load()
        self.device = _dev(device)
        self.lmax = int(lmax)
        self.max_batch = int(max_batch)
        self.n_coeffs = (self.lmax + 1) ** 2
        handle = ctypes.c_void_p()
        with _torch().cuda.device(self.device):
            _lib.check(self.lib.fv_plan_create_points(
                ctypes.byref(handle), self.lmax, self.max_batch, self.device.index))
        self._h = handle

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.fv_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _points(self, xyz):
        torch = _torch()
        if not isinstance(xyz, torch.Tensor) or xyz.dtype != torch.float64 or xyz.dim() != 2 \
                or xyz.shape[1] != 3:
            raise ValueError("xyz must be a (M, 3) float64 tensor")
        if xyz.device != self.device:
            raise ValueError(f"xyz is on {xyz.device}, plan is on {self.device}")
        return xyz.contiguous()

    def forward(self, xyz, w, T, a=None, b=None):
        """Direct-route forward (favest/scalar.py:94-105 + favest/transforms.py:79-147):
        xyz (M, 3) float64 points, w (M,) float64 weights, T (B, M, 3) complex128
        -> (a, b), each (B, (lmax+1)**2) complex128."""
        torch = _torch()
        xyz = self._points(xyz)
        M = int(xyz.shape[0])
        if not isinstance(w, torch.Tensor) or w.dtype != torch.float64 or tuple(w.shape) != (M,):
            raise ValueError(f"w must be a ({M},) float64 tensor")
        if w.device != self.device:
            raise ValueError(f"w is on {w.device}, plan is on {self.device}")
        w = w.contiguous()
        B = int(T.shape[0]) if T.dim() == 3 else -1
        T = _check_tensor(T, (B, M, 3), "T", self.device)
        if a is None:
            a = torch.empty((B, self.n_coeffs), dtype=torch.complex128, device=self.device)
        if b is None:
            b = torch.empty((B, self.n_coeffs), dtype=torch.complex128, device=self.device)
        a = _check_tensor(a, (B, self.n_coeffs), "a", self.device)
        b = _check_tensor(b, (B, self.n_coeffs), "b", self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_forward_points(
                self._h, xyz.data_ptr(), w.data_ptr(), M, T.data_ptr(), a.data_ptr(), b.data_ptr(), B,
                _stream_ptr(self.device)))
        return a, b

    def forward_scalar(self, xyz, w, f, lmax):
        """Direct scalar forward (forward_sht_direct, favest/scalar.py:94-112): xyz (M, 3)
        float64, w (M,) float64, f (B, M) complex128 -> (B, (lmax+1)**2) complex128."""
        torch = _torch()
        xyz = self._points(xyz)
        M = int(xyz.shape[0])
        if not isinstance(w, torch.Tensor) or w.dtype != torch.float64 or tuple(w.shape) != (M,):
            raise ValueError(f"w must be a ({M},) float64 tensor")
        B = int(f.shape[0]) if f.dim() == 2 else -1
        f = _check_tensor(f, (B, M), "f", self.device)
        out = torch.empty((B, (lmax + 1) ** 2), dtype=torch.complex128, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_forward_scalar_points(
                self._h, xyz.data_ptr(), w.contiguous().data_ptr(), M, f.data_ptr(), out.data_ptr(), int(lmax), B,
                _stream_ptr(self.device)))
        return out

    def adjoint_scalar(self, xyz, g, lmax):
        """Direct scalar synthesis (adjoint_sht_direct, favest/scalar.py:115-128):
        xyz (M, 3) float64, g (B, (lmax+1)**2) complex128 -> (B, M) complex128."""
        torch = _torch()
        xyz = self._points(xyz)
        M = int(xyz.shape[0])
        B = int(g.shape[0]) if g.dim() == 2 else -1
        g = _check_tensor(g, (B, (lmax + 1) ** 2), "g", self.device)
        f = torch.empty((B, M), dtype=torch.complex128, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_adjoint_scalar_points(
                self._h, xyz.data_ptr(), M, g.data_ptr(), f.data_ptr(), int(lmax), B, _stream_ptr(self.device)))
        return f

    def adjoint(self, xyz, a, b, T=None):
        """xyz (M, 3) float64, (a, b) (B, K) complex128 -> T (B, M, 3) complex128."""
        torch = _torch()
        xyz = self._points(xyz)
        M = int(xyz.shape[0])
        B = int(a.shape[0]) if a.dim() == 2 else -1
        a = _check_tensor(a, (B, self.n_coeffs), "a", self.device)
        b = _check_tensor(b, (B, self.n_coeffs), "b", self.device)
        if T is None:
            T = torch.empty((B, M, 3), dtype=torch.complex128, device=self.device)
        T = _check_tensor(T, (B, M, 3), "T", self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fv_adjoint_points(
                self._h, xyz.data_ptr(), M, a.data_ptr(), b.data_ptr(), T.data_ptr(), B,
                _stream_ptr(self.device)))
        return T
