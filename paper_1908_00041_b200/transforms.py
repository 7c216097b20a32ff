"""Drop-in ``forward_favest`` / ``adjoint_favest`` on the B200 path.

Same signatures, argument meaning, path selection and error behaviour as the
reference's entry points (``favest/transforms.py:45-181``); the numerics run
in the CUDA library through :mod:`.plan`.  ``tables`` (the reference's
``CGTables``) is accepted for compatibility and only checked for its lmax:
the Clebsch-Gordan factors are evaluated in-kernel with the reference's closed
forms (``favest/coupling.py:39-78``).

Routes (reference: ``_pick_path``, favest/transforms.py:59-76):
  * tensor grid with n_phi >= 2(L+1)+1, path "auto"/"fast-scalar"
      -> ``fv_forward_grid`` / ``fv_adjoint_grid``
  * raw points or "direct-scalar" (adjoint) -> ``fv_adjoint_points``
  * rules without a usable grid, or "direct-scalar" (forward)
      -> ``fv_forward_points`` (favest/scalar.py:94-105)
"""

from __future__ import annotations

import hashlib
import threading
from collections import OrderedDict

import numpy as np

from .core import (
    QuadratureRule,
    ScalarCoefficients,
    TangentFieldSamples,
    VectorCoefficients,
    check_unit,
)
from .grid import TensorGrid

PATHS = ("auto", "direct-scalar", "fast-scalar")

# Plan cache.  Thread safety: _PLANS_LOCK guards the dictionary; every cached
# plan carries a ``call_lock`` that the entry points hold for a whole call
# (upload, kernels, download), because one plan's workspaces serve one call at a
# time (include/favest_b200.h).  Evicted or outgrown plans are only dropped from
# the cache, never closed here: a caller may still hold one (grid_plan() /
# points_plan() are public), and the plan frees its device memory when the
# last reference goes.
_PLANS: "OrderedDict[tuple, object]" = OrderedDict()
_PLANS_LOCK = threading.Lock()
_MAX_PLANS = 8


def _resolve_grid(rule_or_points):
    """(points, grid, rule) from a rule / grid / raw (N, 3) array
    (favest/transforms.py:49-56); duck-typed so reference instances work."""
    if hasattr(rule_or_points, "weights") and hasattr(rule_or_points, "points"):
        return np.asarray(rule_or_points.points, dtype=np.float64), getattr(rule_or_points, "grid", None), rule_or_points
    if hasattr(rule_or_points, "ring_thetas") and hasattr(rule_or_points, "n_phi"):
        return rule_or_points.points(), rule_or_points, None
    pts = check_unit(np.atleast_2d(np.asarray(rule_or_points, dtype=np.float64)))
    return pts, None, None


def _pick_path(path: str, grid, lmax: int) -> bool:
    """True for the grid (fast) route (favest/transforms.py:59-76)."""
    if path not in PATHS:
        raise ValueError(f"unknown path {path!r}; expected one of {PATHS}")
    needed = 2 * (lmax + 1) + 1
    usable = grid is not None and grid.n_phi >= needed
    if path == "fast-scalar":
        if grid is None:
            raise ValueError("fast-scalar path requires a rule with tensor-grid structure")
        if grid.n_phi < needed:
            raise ValueError(
                f"fast-scalar path needs n_phi >= {needed} for degree {lmax}, "
                f"grid has n_phi={grid.n_phi}"
            )
        return True
    if path == "direct-scalar":
        return False
    return usable


def _grid_key(grid, lmax, device):
    th = np.ascontiguousarray(grid.ring_thetas, dtype=np.float64)
    w = np.ascontiguousarray(grid.ring_weights, dtype=np.float64)
    h = hashlib.blake2b(th.tobytes() + w.tobytes(), digest_size=16).hexdigest()
    return ("grid", int(lmax), int(grid.n_phi), th.size, h, str(device))


def _cached(key, make, batch):
    with _PLANS_LOCK:
        plan = _PLANS.get(key)
        if plan is None or plan.max_batch < batch:
            plan = make(max(batch, plan.max_batch if plan is not None else 1))
            plan.call_lock = threading.Lock()
            _PLANS[key] = plan
        _PLANS.move_to_end(key)
        while len(_PLANS) > _MAX_PLANS:
            _PLANS.popitem(last=False)
        return plan


def grid_plan(grid, lmax, batch=1, device=None):
    """Cached :class:`GridPlan` for (grid, lmax, device) with capacity >= batch."""
    from .plan import GridPlan, _dev

    dev = _dev(device)
    return _cached(_grid_key(grid, lmax, dev),
                   lambda mb: GridPlan.from_grid(grid, lmax, max_batch=mb, device=dev), batch)


def points_plan(lmax, batch=1, device=None):
    from .plan import PointsPlan, _dev

    dev = _dev(device)
    return _cached(("points", int(lmax), str(dev)),
                   lambda mb: PointsPlan(lmax, max_batch=mb, device=dev), batch)


def _to_device(arr: np.ndarray, device):
    """Host array -> device tensor through the pipelined pinned stager (staging.py)."""
    from .staging import stager

    return stager(device).to_device(arr)


def _to_host(x) -> np.ndarray:
    """Device tensor -> new pageable numpy array through the pipelined pinned stager."""
    from .staging import stager

    return stager(x.device).to_host(x)


def _check_tables(tables, lmax):
    if tables is not None and getattr(tables, "lmax", lmax) < lmax:
        raise ValueError(f"tables built for lmax={tables.lmax} cannot serve lmax={lmax}")


def forward_favest(samples, rule, lmax: int, path: str = "auto", tables=None) -> VectorCoefficients:
    """Forward VSHT: tangent samples at the rule's points -> div/curl coefficients
    for 1 <= l <= lmax (favest/transforms.py:79-147)."""
    import torch

    if lmax < 1:
        raise ValueError(f"vector transforms need lmax >= 1, got {lmax}")
    spts = np.asarray(samples.points)
    rpts = np.asarray(rule.points)
    # samples built on the rule's own point array (the usual case) need no O(N) check
    if spts is not rpts and (spts.shape != rpts.shape or not (
            np.array_equal(spts, rpts) or np.allclose(spts, rpts, rtol=0.0, atol=1e-12))):
        raise ValueError("sample points do not match the quadrature rule points")
    grid = getattr(rule, "grid", None)
    use_fast = _pick_path(path, grid, lmax)
    _check_tables(tables, lmax)
    vals = np.ascontiguousarray(samples.values, dtype=np.complex128).reshape(1, -1, 3)
    plan = grid_plan(grid, lmax) if use_fast else points_plan(lmax)
    with plan.call_lock, torch.cuda.device(plan.device):
        if use_fast:
            a, b = plan.forward(_to_device(vals, plan.device))
        else:  # direct route on the rule's own points and weights (favest/scalar.py:94-105)
            xyz = _to_device(np.ascontiguousarray(rpts, dtype=np.float64), plan.device)
            w = _to_device(np.ascontiguousarray(rule.weights, dtype=np.float64), plan.device)
            a, b = plan.forward(xyz, w, _to_device(vals, plan.device))
        a = _to_host(a[0])
        b = _to_host(b[0])
    return VectorCoefficients(ScalarCoefficients._trusted(lmax, a), ScalarCoefficients._trusted(lmax, b))


def adjoint_favest(coeffs, rule_or_points, path: str = "auto", tables=None) -> TangentFieldSamples:
    """Adjoint VSHT: coefficients -> tangent field at a rule / grid / raw points
    (favest/transforms.py:150-181)."""
    import torch

    points, grid, _ = _resolve_grid(rule_or_points)
    lmax = coeffs.lmax
    use_fast = _pick_path(path, grid, lmax)
    _check_tables(tables, lmax)
    a = np.ascontiguousarray(coeffs.div.values, dtype=np.complex128).reshape(1, -1)
    b = np.ascontiguousarray(coeffs.curl.values, dtype=np.complex128).reshape(1, -1)
    plan = grid_plan(grid, lmax) if use_fast else points_plan(lmax)
    with plan.call_lock, torch.cuda.device(plan.device):
        a_d, b_d = _to_device(a, plan.device), _to_device(b, plan.device)
        if use_fast:
            T = plan.adjoint(a_d, b_d)
        else:
            T = plan.adjoint(_to_device(np.ascontiguousarray(points, dtype=np.float64), plan.device), a_d, b_d)
        values = _to_host(T[0])
    # points came from a validated rule / grid, or were checked by _resolve_grid
    return TangentFieldSamples._trusted(points, values)


__all__ = [
    "PATHS", "forward_favest", "adjoint_favest", "grid_plan", "points_plan",
    "TensorGrid", "QuadratureRule",
]
