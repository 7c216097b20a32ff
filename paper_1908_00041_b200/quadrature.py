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


# favest/data/icosahedron12.txt, in file order: the two coordinates as the
# data file spells them (17 significant digits); row k is the sign triple
# _ICO_ROWS[k] times the magnitudes (0, A, B), (A, B, 0), (B, 0, A) for k mod 3.
_ICO_A = 0.52573111211913359
_ICO_B = 0.85065080835203999
_ICO_ROWS = (
    (0, 1, 1), (1, 1, 0), (1, 0, 1), (0, 1, -1), (1, -1, 0), (-1, 0, 1),
    (0, -1, 1), (-1, 1, 0), (1, 0, -1), (0, -1, -1), (-1, -1, 0), (-1, 0, -1),
)


def _icosahedron() -> np.ndarray:
    """The reference's bundled 12-point design, row for row, through the same
    renormalisation as load_design (favest/quadrature.py:79-109,134-139)."""
    pattern = ((0.0, _ICO_A, _ICO_B), (_ICO_A, _ICO_B, 0.0), (_ICO_B, 0.0, _ICO_A))
    rows = [[sg * mag for sg, mag in zip(signs, pattern[k % 3])] for k, signs in enumerate(_ICO_ROWS)]
    return renormalize(np.array(rows, dtype=np.float64), "icosahedron12.txt")


_BUNDLED = {"icosahedron12": (_icosahedron, 5)}


def bundled_design(name: str = "icosahedron12") -> QuadratureRule:
    """A design shipped with the package (favest/quadrature.py:100-109): the
    icosahedron has the reference data file's rows, order and values."""
    try:
        make, t = _BUNDLED[name]
    except KeyError:
        raise ValueError(f"unknown bundled design {name!r}; available: {sorted(_BUNDLED)}") from None
    pts = make()
    n = pts.shape[0]
    return QuadratureRule(points=pts, weights=np.full(n, FOUR_PI / n), exactness=t, kind="spherical-design")


__all__ = ["gen_gl_tensor", "verify_exactness", "load_design", "bundled_design"]
