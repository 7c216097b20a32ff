"""Iso-latitude tensor grids — the host-side input provider of the GPU path.

``TensorGrid`` mirrors ``favest/scalar.py:29-84`` and ``gen_gl_tensor`` mirrors
``favest/quadrature.py:29-48``.  The ring colatitudes and weights are handed to
the device verbatim (``fv_plan_create_grid``): the reference's scipy
Gauss-Legendre polar weights carry a 1e-10..2e-7 relative error (SURVEY
§0.6), so parity requires the very same arrays, never a recomputation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import QuadratureRule, from_spherical


@dataclass
class TensorGrid:
    """Ring colatitudes (strictly increasing in (0, pi)), per-point ring weights
    (including 2 pi / n_phi) and n_phi equispaced longitudes; ring-major points."""

    ring_thetas: np.ndarray
    ring_weights: np.ndarray
    n_phi: int

    def __post_init__(self) -> None:
        th = np.atleast_1d(np.asarray(self.ring_thetas, dtype=np.float64))
        w = np.atleast_1d(np.asarray(self.ring_weights, dtype=np.float64))
        if th.ndim != 1 or th.shape != w.shape:
            raise ValueError("ring_thetas and ring_weights must be matching 1-d arrays")
        if th.size == 0:
            raise ValueError("grid needs at least one ring")
        if np.any(th <= 0.0) or np.any(th >= np.pi):
            raise ValueError("ring colatitudes must lie strictly inside (0, pi)")
        if np.any(np.diff(th) <= 0.0):
            raise ValueError("ring colatitudes must be strictly increasing")
        if self.n_phi < 1:
            raise ValueError(f"n_phi must be positive, got {self.n_phi}")
        self.ring_thetas = th
        self.ring_weights = w

    @property
    def n_theta(self) -> int:
        return self.ring_thetas.size

    def __len__(self) -> int:
        return self.n_theta * self.n_phi

    @property
    def phis(self) -> np.ndarray:
        return 2.0 * np.pi * np.arange(self.n_phi) / self.n_phi

    def points(self) -> np.ndarray:
        theta = np.repeat(self.ring_thetas, self.n_phi)
        phi = np.tile(self.phis, self.n_theta)
        return from_spherical(theta, phi)

    def to_rule(self, exactness: int, kind: str = "gl-tensor") -> QuadratureRule:
        return QuadratureRule(
            points=self.points(),
            weights=np.repeat(self.ring_weights, self.n_phi),
            exactness=exactness,
            kind=kind,
            grid=self,
        )


def gen_gl_tensor(t: int, on_device: bool = False) -> tuple[TensorGrid, QuadratureRule]:
    """Gauss-Legendre tensor rule exact to degree t (favest/quadrature.py:29-48):
    (t+2)//2 rings, t+1 longitudes, weights (2 pi / n_phi) * gauss weight.

    Default: scipy's roots_legendre, as the reference (bitwise its weights).
    ``on_device=True``: the rule from the CUDA library (fv_gauss_legendre: Newton
    on the colatitudes, the Legendre recurrence in difference form on
    1 - cos(theta), ring colatitudes without an arccos), a deliberate deviation:
    polar weights accurate to ~1e-11 where scipy's are off by 1e-9 .. 1e-7, and
    an exactness defect of ~1e-14 against scipy's ~4e-13 at n = 4098 (SURVEY
    §0.6; tests/test_gpu_edges.py), so not bitwise the reference's rule."""
    if t < 0:
        raise ValueError(f"exactness degree must be non-negative, got {t}")
    n_theta = (t + 2) // 2
    n_phi = t + 1
    if on_device:
        thetas, gauss_w = gauss_legendre_device(n_theta)
        weights = gauss_w * (2.0 * np.pi / n_phi)
    else:
        from scipy.special import roots_legendre

        nodes, gauss_w = roots_legendre(n_theta)
        thetas = np.arccos(nodes[::-1])
        weights = gauss_w[::-1] * (2.0 * np.pi / n_phi)
    grid = TensorGrid(ring_thetas=thetas, ring_weights=weights, n_phi=n_phi)
    return grid, grid.to_rule(exactness=t)


def gauss_legendre_device(n: int, device=None) -> tuple[np.ndarray, np.ndarray]:
    """(colatitudes ascending, Gauss weights) of the n-node rule, computed on the GPU."""
    import ctypes

    import torch

    from . import _lib

    if not torch.cuda.is_available():
        raise RuntimeError("gauss_legendre_device needs a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    th = np.empty(int(n), dtype=np.float64)
    w = np.empty(int(n), dtype=np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    lib = _lib.load()
    _lib.check(lib.fv_gauss_legendre(int(n), th.ctypes.data_as(dp), w.ctypes.data_as(dp), int(dev)))
    return th, w


def gl_grid_for(lmax: int) -> tuple[TensorGrid, QuadratureRule]:
    """The BASELINE grid for vector degree lmax: gen_gl_tensor(2*lmax+3) ->
    n_theta = lmax+2 rings, n_phi = 2*lmax+4."""
    return gen_gl_tensor(2 * lmax + 3)
