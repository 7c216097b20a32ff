"""Scalar spherical harmonic transforms and rule certification on the B200 path.

Same signatures, argument meaning and errors as the reference's public scalar
functions (``favest/scalar.py:108-184``) and ``verify_exactness``
(``favest/quadrature.py:51-76``); the numerics run in the CUDA library
(``fv_forward_scalar_grid`` / ``fv_adjoint_scalar_grid`` /
``fv_forward_scalar_points`` / ``fv_adjoint_scalar_points``): the scalar
fields ride as the Cartesian components of pseudo fields through the same
ring DFTs, folded Legendre contractions and scattered-point kernels as the
vector transforms.  A plan of vector degree L serves scalar degrees <= L + 1,
so scalar degree lmax uses L = max(1, lmax - 1); on a tensor grid that needs
n_phi >= 2 max(lmax, 2) + 1.
"""

from __future__ import annotations

import numpy as np

from .core import FOUR_PI, ScalarCoefficients, check_unit
from .transforms import _to_device, _to_host, grid_plan, points_plan


def _plan_degree(lmax: int) -> int:
    return max(1, int(lmax) - 1)


def _values(f, n):
    vals = np.asarray(f, dtype=np.complex128)
    if vals.shape[0] != n or vals.ndim not in (1, 2):  # favest/scalar.py:87-91
        raise ValueError(f"sample array of shape {vals.shape} does not match {n} points")
    return vals


def _require_bandwidth(grid, lmax: int) -> None:  # favest/scalar.py:139-143
    if grid.n_phi < 2 * lmax + 1:
        raise ValueError(
            f"fast path needs n_phi >= 2*lmax+1 = {2 * lmax + 1}, grid has n_phi={grid.n_phi}"
        )


class _GridRule:
    """points / weights of a tensor grid, ring-major (favest/scalar.py:72-84)"""

    def __init__(self, grid):
        self.points = grid.points()
        self.weights = np.repeat(np.asarray(grid.ring_weights, dtype=np.float64), grid.n_phi)


def _columns(vals):
    """(n,) or (n, c) complex -> torch (c, n) on the host"""
    import torch

    cols = vals[:, None] if vals.ndim == 1 else vals
    return torch.from_numpy(np.ascontiguousarray(cols.T))


def forward_sht_fast(f, grid, lmax: int) -> ScalarCoefficients:
    """Forward scalar transform on a tensor grid (favest/scalar.py:157-167)."""
    if lmax < 0:
        raise ValueError(f"lmax must be non-negative, got {lmax}")
    _require_bandwidth(grid, lmax)
    vals = _values(f, grid.n_theta * grid.n_phi)
    if grid.n_phi < 2 * (_plan_degree(lmax) + 1) + 1:
        # lmax <= 1 on a 3- or 4-point ring: below the vector plan's bandwidth,
        # and alias-free, so the direct sum over the flattened grid is the same map
        return forward_sht_direct(vals, _GridRule(grid), lmax)
    plan = grid_plan(grid, _plan_degree(lmax))
    cols = _columns(vals)
    out = np.concatenate([_to_host(plan.forward_scalar(_to_device(c.numpy(), plan.device), lmax))
                          for c in cols.split(3 * plan.max_batch)])
    values = out.T if vals.ndim == 2 else out[0]
    return ScalarCoefficients(lmax, values)


def adjoint_sht_fast(coeffs: ScalarCoefficients, grid) -> np.ndarray:
    """Harmonic partial sum on a tensor grid (favest/scalar.py:182-184)."""
    lmax = coeffs.lmax
    _require_bandwidth(grid, lmax)
    if grid.n_phi < 2 * (_plan_degree(lmax) + 1) + 1:
        return adjoint_sht_direct(coeffs, grid.points())
    plan = grid_plan(grid, _plan_degree(lmax))
    import torch

    g = torch.from_numpy(np.ascontiguousarray(np.asarray(coeffs.values, dtype=np.complex128)[None]))
    return _to_host(plan.adjoint_scalar(g.to(plan.device), lmax)[0])


def forward_sht_direct(f, rule, lmax: int) -> ScalarCoefficients:
    """Forward scalar transform by direct summation over the rule's points
    (favest/scalar.py:108-112)."""
    import torch

    if lmax < 0:
        raise ValueError(f"lmax must be non-negative, got {lmax}")
    pts = np.asarray(rule.points, dtype=np.float64)
    vals = _values(f, pts.shape[0])
    plan = points_plan(_plan_degree(lmax))
    xyz = torch.from_numpy(np.ascontiguousarray(pts)).to(plan.device)
    w = torch.from_numpy(np.ascontiguousarray(rule.weights, dtype=np.float64)).to(plan.device)
    cols = _columns(vals)
    out = np.concatenate([_to_host(plan.forward_scalar(xyz, w, _to_device(c.numpy(), plan.device), lmax))
                          for c in cols.split(3 * plan.max_batch)])
    values = out.T if vals.ndim == 2 else out[0]
    return ScalarCoefficients(lmax, values)


def adjoint_sht_direct(coeffs: ScalarCoefficients, points) -> np.ndarray:
    """Harmonic partial sum at arbitrary points (favest/scalar.py:115-117)."""
    import torch

    pts = check_unit(np.atleast_2d(np.asarray(points, dtype=np.float64)))
    lmax = coeffs.lmax
    plan = points_plan(_plan_degree(lmax))
    xyz = torch.from_numpy(np.ascontiguousarray(pts)).to(plan.device)
    g = torch.from_numpy(np.ascontiguousarray(np.asarray(coeffs.values, dtype=np.complex128)[None]))
    return _to_host(plan.adjoint_scalar(xyz, g.to(plan.device), lmax)[0])


def verify_exactness(rule, t: int) -> tuple[float, bool]:
    """Certify that a rule integrates all harmonics of degree <= t
    (favest/quadrature.py:51-76): the largest |sum_i w_i Y(l, m, x_i) -
    sqrt(4 pi) [l = m = 0]| over l <= t, |m| <= l (real weights: the m >= 0
    half suffices), passed if <= 1e-8.  The sums are the direct forward
    transform of the constant 1 (conj(Y) and Y give the same moduli)."""
    if t < 0:
        raise ValueError(f"certification degree must be non-negative, got {t}")
    n = np.asarray(rule.points).shape[0]
    c = forward_sht_direct(np.ones(n, dtype=np.complex128), rule, t).values
    ms = np.concatenate([np.arange(-l, l + 1) for l in range(t + 1)])
    sums = c[ms >= 0].copy()
    sums[0] -= np.sqrt(FOUR_PI)
    defect = float(np.max(np.abs(sums)))
    return defect, defect <= 1e-8


__all__ = ["forward_sht_fast", "adjoint_sht_fast", "forward_sht_direct", "adjoint_sht_direct", "verify_exactness"]
