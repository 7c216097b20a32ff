"""Quadrature rules around the transforms (favest/quadrature.py:29-109):
Gauss-Legendre tensor rules, spherical designs from files, the bundled
icosahedron, and rule certification on the GPU."""

from __future__ import annotations

import numpy as np

from .core import FOUR_PI, QuadratureRule
from .grid import gen_gl_tensor
from .io import read_columns, renormalize
from .scalar import verify_exactness


def load_design(path, t: int) -> QuadratureRule:
    """Equal-weight spherical design from a 3-column text file
    (favest/quadrature.py:79-97): points off the unit sphere by more than
    1e-6 are rejected, smaller deviations renormalised, weights 4 pi / N."""
    raw = read_columns(path)
    if raw.shape[1] != 3:
        raise ValueError(f"design file must have 3 columns, found {raw.shape[1]} in {path}")
    points = renormalize(raw, path)
    n = points.shape[0]
    return QuadratureRule(points=points, weights=np.full(n, FOUR_PI / n), exactness=t, kind="spherical-design")


def _icosahedron() -> np.ndarray:
    """The 12 vertices (0, +-1, +-phi) and cyclic permutations, on the unit sphere."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    base = []
    for s1 in (1.0, -1.0):
        for s2 in (1.0, -1.0):
            base.append((0.0, s1, s2 * phi))
    pts = []
    for k in range(3):
        for v in base:
            pts.append(np.roll(v, k))
    pts = np.array(pts)
    return pts / np.linalg.norm(pts, axis=1, keepdims=True)


_BUNDLED = {"icosahedron12": (_icosahedron, 5)}


def bundled_design(name: str = "icosahedron12") -> QuadratureRule:
    """A design shipped with the package (favest/quadrature.py:100-109); the
    icosahedron is generated from its closed form (vertex order may differ
    from the reference's data file; the set is the same to 1 ulp)."""
    try:
        make, t = _BUNDLED[name]
    except KeyError:
        raise ValueError(f"unknown bundled design {name!r}; available: {sorted(_BUNDLED)}") from None
    pts = make()
    n = pts.shape[0]
    return QuadratureRule(points=pts, weights=np.full(n, FOUR_PI / n), exactness=t, kind="spherical-design")


__all__ = ["gen_gl_tensor", "verify_exactness", "load_design", "bundled_design"]
