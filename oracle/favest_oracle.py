"""TEST INFRASTRUCTURE ONLY — numpy restatement of the FaVeST VSHT hot path.

Every function cites the reference file:line it follows (paths relative to
``/root/reference/pkg/src/favest/``).  This module is the *checker* for the
CUDA path and the ``port`` CPU baseline in ``bench.py``; it is never imported
by ``paper_1908_00041_b200``.

Differences from the literal reference, all deliberate:

* Streaming per order m (O(n_theta * L) memory instead of the reference's
  dense ``legendre_table`` / fancy-gather temporaries, which need ~112 GB at
  L=1024 and ~275 GB at L=4096).
* Extended-range ("X-number") seeds and recurrence: the diagonal seed
  ``Pbar_m^m ~ sin^m(theta)`` is carried as ``x * 2**e`` with ``e`` a
  multiple of 512, so it cannot underflow.  Power-of-two rescaling is exact,
  so wherever the reference stays in the normal double range the Legendre
  values are *bitwise* equal to ``legendre_table`` (checked in
  ``tests/test_oracle.py`` against golden vectors); where the reference
  underflows (L >~ 1900) it returns the true values instead of 0/NaN.
  Values whose scaled exponent is below -1024 (magnitude < 2**-512 * 2**-512)
  are returned as 0.
* Summation order of the contractions (BLAS instead of einsum).
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "FOUR_PI", "INV_SQRT_4PI", "INV_SQRT2", "flat_size", "degrees_orders", "tri_index",
    "gl_grid", "grid_points", "ring_cos_sin", "seed_table", "recurrence_ab", "legendre_m",
    "legendre_table", "sht_forward_grid", "sht_adjoint_grid", "forward_order", "adjoint_order", "sht_adjoint_points",
    "sht_forward_points", "vsht_forward_points", "verify_exactness",
    "cg_explicit_vec", "cg_tables", "shift_read", "vsht_forward_grid", "vsht_adjoint_merged",
    "vsht_adjoint_grid", "vsht_adjoint_points", "coef", "random_points", "tangent_noise",
    "rel_l2", "XR_SHIFT",
]

# favest/core.py:17 and favest/legendre.py:24
FOUR_PI = 4.0 * np.pi
INV_SQRT_4PI = 1.0 / np.sqrt(FOUR_PI)
# favest/transforms.py:46
INV_SQRT2 = 1.0 / np.sqrt(2.0)

#: exponent step of the extended-range representation value = x * 2**e
XR_SHIFT = 512
_XR_BIG = 2.0 ** XR_SHIFT
_XR_SMALL = 2.0 ** -XR_SHIFT


# --------------------------------------------------------------------------
# layout — favest/core.py:23-56, favest/legendre.py:27-33
# --------------------------------------------------------------------------

def flat_size(lmax: int) -> int:
    """favest/core.py:40-44 — (lmax+1)**2 pairs (l, m), flat index l*l+l+m."""
    return (lmax + 1) ** 2


def degrees_orders(lmax: int) -> tuple[np.ndarray, np.ndarray]:
    """favest/core.py:47-56 — (ls, ms) in flat degree-major order."""
    k = np.arange(flat_size(lmax), dtype=np.int64)
    ls = np.floor(np.sqrt(k)).astype(np.int64)
    # guard the float sqrt at perfect squares
    ls = np.where((ls + 1) ** 2 <= k, ls + 1, ls)
    ls = np.where(ls * ls > k, ls - 1, ls)
    ms = k - ls * ls - ls
    return ls, ms


def tri_index(l, m):
    """favest/legendre.py:27-29."""
    return l * (l + 1) // 2 + m


# --------------------------------------------------------------------------
# grid — favest/quadrature.py:29-48, favest/scalar.py:29-84
# --------------------------------------------------------------------------

def gl_grid(lmax: int):
    """The BASELINE grid ``gen_gl_tensor(2*lmax+3)`` (favest/quadrature.py:29-48).

    Returns (ring_thetas, ring_weights, n_phi) with n_theta = lmax+2 rings and
    n_phi = 2*lmax+4; weights include the 2*pi/n_phi longitude factor.  The
    scipy call is the same one the reference makes, so weights are bitwise
    the reference's (including scipy's polar-weight error).
    """
    from scipy.special import roots_legendre

    t = 2 * lmax + 3
    n_theta = (t + 2) // 2
    n_phi = t + 1
    nodes, gauss_w = roots_legendre(n_theta)
    thetas = np.arccos(nodes[::-1])
    weights = gauss_w[::-1] * (2.0 * np.pi / n_phi)
    return np.ascontiguousarray(thetas), np.ascontiguousarray(weights), n_phi


def grid_points(ring_thetas, n_phi):
    """favest/scalar.py:66-74 + favest/core.py:86-91 — ring-major unit points."""
    theta = np.repeat(np.asarray(ring_thetas, dtype=np.float64), n_phi)
    phis = 2.0 * np.pi * np.arange(n_phi) / n_phi
    phi = np.tile(phis, len(ring_thetas))
    st = np.sin(theta)
    return np.stack([st * np.cos(phi), st * np.sin(phi), np.cos(theta)], axis=-1)


def ring_cos_sin(ring_thetas):
    """t = clip(cos theta), s = sqrt(max(0, 1-t*t)) — favest/scalar.py:133,
    favest/legendre.py:53-57."""
    t = np.clip(np.cos(np.asarray(ring_thetas, dtype=np.float64)), -1.0, 1.0)
    s = np.sqrt(np.maximum(0.0, 1.0 - t * t))
    return t, s


# --------------------------------------------------------------------------
# normalized associated Legendre functions — favest/legendre.py:36-75
# --------------------------------------------------------------------------

def seed_table(lt: int, s: np.ndarray):
    """Extended-range diagonal seeds Pbar_m^m for m = 0..lt.

    favest/legendre.py:60-65: Pbar_0^0 = 1/sqrt(4 pi);
    Pbar_m^m = (-sqrt((2m+1)/(2m)) * s) * Pbar_{m-1}^{m-1}, evaluated in that
    operation order.  Returns (x, e) of shape (lt+1, n) with value x * 2**e.
    """
    s = np.asarray(s, dtype=np.float64)
    x = np.empty((lt + 1,) + s.shape)
    e = np.zeros((lt + 1,) + s.shape, dtype=np.int64)
    cur = np.full(s.shape, INV_SQRT_4PI)
    cur_e = np.zeros(s.shape, dtype=np.int64)
    x[0] = cur
    for m in range(1, lt + 1):
        cur = -np.sqrt((2 * m + 1) / (2.0 * m)) * s * cur
        small = (np.abs(cur) < _XR_SMALL) & (cur != 0.0)
        if np.any(small):
            cur = np.where(small, cur * _XR_BIG, cur)
            cur_e = np.where(small, cur_e - XR_SHIFT, cur_e)
        x[m] = cur
        e[m] = cur_e
    return x, e


def recurrence_ab(m: int, lt: int):
    """Coefficients a_l, b_l for l = m+2..lt (favest/legendre.py:70-71), same
    expression order, so bitwise equal to the reference's."""
    l = np.arange(m + 2, lt + 1, dtype=np.int64)
    lf = l.astype(np.float64)
    a = np.sqrt((4.0 * lf * lf - 1.0) / (l * l - m * m).astype(np.float64))
    lm1 = lf - 1.0
    b = np.sqrt((lm1 * lm1 - float(m * m)) / (4.0 * (lm1 * lm1) - 1.0))
    return a, b


def _xr_value(p, e):
    """value = p * 2**e; exponents below -1024 flush to 0 (see module doc)."""
    out = np.ldexp(p, e.astype(np.int32) if hasattr(e, "astype") else int(e))
    return np.where(e < -2 * XR_SHIFT, 0.0, out)


def legendre_m(m: int, lt: int, t: np.ndarray, seed_x: np.ndarray, seed_e: np.ndarray) -> np.ndarray:
    """Rows Pbar_l^m(t) for l = m..lt, shape (lt+1-m, n).

    favest/legendre.py:66-74: Pbar_{m+1}^m = (sqrt(2m+3) * t) * Pbar_m^m, then
    Pbar_l^m = a * (t * Pbar_{l-1}^m - b * Pbar_{l-2}^m), in extended range.
    """
    t = np.asarray(t, dtype=np.float64)
    n_l = lt + 1 - m
    out = np.empty((n_l,) + t.shape)
    p2 = seed_x.copy()
    e = seed_e.copy()
    scaled = bool(np.any(e < 0))
    out[0] = _xr_value(p2, e) if scaled else p2
    if n_l == 1:
        return out
    p1 = np.sqrt(2 * m + 3.0) * t * p2
    out[1] = _xr_value(p1, e) if scaled else p1
    if n_l == 2:
        return out
    a, b = recurrence_ab(m, lt)
    for i in range(n_l - 2):
        p = a[i] * (t * p1 - b[i] * p2)
        p2, p1 = p1, p
        if scaled:
            big = (e < 0) & (np.abs(p1) >= _XR_BIG)
            if np.any(big):
                p1 = np.where(big, p1 * _XR_SMALL, p1)
                p2 = np.where(big, p2 * _XR_SMALL, p2)
                e = np.where(big, e + XR_SHIFT, e)
            out[i + 2] = _xr_value(p1, e)
            if not np.any(e < 0):
                scaled = False
        else:
            out[i + 2] = p1
    return out


def legendre_table(lmax: int, t: np.ndarray) -> np.ndarray:
    """Same contract as favest/legendre.py:36-75 (packed triangle, column
    tri_index(l, m)), built from the extended-range per-order rows."""
    t = np.clip(np.asarray(t, dtype=np.float64), -1.0, 1.0)
    s = np.sqrt(np.maximum(0.0, 1.0 - t * t))
    sx, se = seed_table(lmax, s)
    out = np.empty(t.shape + ((lmax + 1) * (lmax + 2) // 2,))
    for m in range(lmax + 1):
        rows = legendre_m(m, lmax, t, sx[m], se[m])
        ls = np.arange(m, lmax + 1)
        out[..., tri_index(ls, m)] = np.moveaxis(rows, 0, -1)
    return out


# --------------------------------------------------------------------------
# scalar transforms — favest/scalar.py:120-128, 146-154, 170-179
# --------------------------------------------------------------------------

def _sigma(m: int) -> float:
    """favest/legendre.py:101-103 — (-1)**m for m < 0, +1 otherwise."""
    return 1.0 if (m >= 0 or (-m) % 2 == 0) else -1.0


def sht_forward_grid(f, ring_thetas, ring_weights, n_phi, lt, orders=None):
    """Scalar forward on a tensor grid (favest/scalar.py:146-154).

    F_{l,m} = sigma_m * sum_r Pbar_l^{|m|}(t_r) * w_r * fft(f_r)[m mod n_phi].
    ``f`` is (N, C) complex, ring-major.  Returns (flat_size(lt), C).  If
    ``orders`` is given only those |m| are computed (others left 0).
    """
    f = np.asarray(f, dtype=np.complex128)
    n_theta = len(ring_thetas)
    C = f.shape[1]
    spec = np.fft.fft(f.reshape(n_theta, n_phi, C), axis=1)  # scalar.py:149
    w = np.asarray(ring_weights, dtype=np.float64)
    t, s = ring_cos_sin(ring_thetas)
    sx, se = seed_table(lt, s)
    out = np.zeros((flat_size(lt), C), dtype=np.complex128)
    ms_iter = range(lt + 1) if orders is None else sorted(set(int(x) for x in orders))
    for m in ms_iter:
        for mm, rows in forward_order(m, spec, w, t, sx, se, lt):
            ls = np.arange(m, lt + 1)
            out[ls * ls + ls + mm] = rows
    return out


def forward_order(m, spec, w, t, sx, se, lt):
    """The per-order stage of sht_forward_grid (favest/scalar.py:150-153) from
    the ring spectra ``spec`` (n_theta, n_phi, C): [(+m, rows), (-m, rows)] with
    rows (lt+1-m, C) = sigma_m * sum_r Pbar_l^m(t_r) w_r spec[r, m mod n_phi]."""
    n_phi = spec.shape[1]
    P = legendre_m(m, lt, t, sx[m], se[m])  # (n_l, n_theta)
    res = []
    for sgn in ((1,) if m == 0 else (1, -1)):
        mm = sgn * m
        g = w[:, None] * spec[:, mm % n_phi, :]  # scalar.py:151-152
        res.append((mm, _sigma(mm) * (P @ g.real + 1j * (P @ g.imag))))
    return res


def sht_adjoint_grid(g, lt, ring_thetas, n_phi, orders=None, spectrum=False):
    """Scalar adjoint on a tensor grid (favest/scalar.py:170-179):
    spectrum[r, m mod n_phi] = sum_l Pbar_l^{|m|}(t_r) sigma_m g_{l,m}, then
    ifft * n_phi.  ``g`` is (flat_size(lt), C).  Returns (N, C)."""
    g = np.asarray(g, dtype=np.complex128)
    n_theta = len(ring_thetas)
    C = g.shape[1]
    if n_phi < 2 * lt + 1:  # scalar.py:139-143
        raise ValueError(
            f"fast path needs n_phi >= 2*lmax+1 = {2 * lt + 1}, grid has n_phi={n_phi}"
        )
    t, s = ring_cos_sin(ring_thetas)
    sx, se = seed_table(lt, s)
    spec = np.zeros((n_theta, n_phi, C), dtype=np.complex128)
    ms_iter = range(lt + 1) if orders is None else sorted(set(int(x) for x in orders))
    for m in ms_iter:
        for mm, col in adjoint_order(m, g, t, sx, se, lt):
            spec[:, mm % n_phi, :] = col
    if spectrum:  # ring spectra before the inverse DFT: (n_theta, n_phi, C)
        return spec
    out = np.fft.ifft(spec, axis=1) * n_phi
    return out.reshape(n_theta * n_phi, C)


def adjoint_order(m, g, t, sx, se, lt):
    """The per-order stage of sht_adjoint_grid (favest/scalar.py:174-176):
    [(+m, bins), (-m, bins)] with bins (n_theta, C) = sum_l Pbar_l^m(t_r)
    sigma_m g_{l,m}."""
    P = legendre_m(m, lt, t, sx[m], se[m])  # (n_l, n_theta)
    ls = np.arange(m, lt + 1)
    res = []
    for sgn in ((1,) if m == 0 else (1, -1)):
        mm = sgn * m
        cols = _sigma(mm) * g[ls * ls + ls + mm]  # (n_l, C)
        res.append((mm, P.T @ cols.real + 1j * (P.T @ cols.imag)))
    return res


def sht_adjoint_points(g, lt, points):
    """Scalar adjoint at scattered points (favest/scalar.py:120-128 with
    ylm_table, favest/legendre.py:106-123): f(x_p) = sum g_{l,m} Y_{l,m}(x_p),
    t_p = z_p, phi_p = atan2(y_p, x_p) mod 2 pi (favest/core.py:74-83)."""
    g = np.asarray(g, dtype=np.complex128)
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    C = g.shape[1]
    z = np.clip(pts[:, 2], -1.0, 1.0)
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = np.mod(np.arctan2(pts[:, 1], pts[:, 0]), 2.0 * np.pi)
    sx, se = seed_table(lt, s)
    out = np.zeros((pts.shape[0], C), dtype=np.complex128)
    for m in range(lt + 1):
        P = legendre_m(m, lt, z, sx[m], se[m])  # (n_l, M)
        ls = np.arange(m, lt + 1)
        for sgn in ((1,) if m == 0 else (1, -1)):
            mm = sgn * m
            cols = _sigma(mm) * g[ls * ls + ls + mm]
            acc = P.T @ cols.real + 1j * (P.T @ cols.imag)  # (M, C)
            out += np.exp(1j * mm * phi)[:, None] * acc
    return out


def sht_forward_points(f, weights, points, lt):
    """Scalar forward by direct summation over arbitrary weighted points
    (favest/scalar.py:94-105 with ylm_table, favest/legendre.py:106-123):
    F_{l,m} = sum_k w_k f_k conj(Y_{l,m}(x_k)),
    conj(Y_{l,m}) = sigma_m Pbar_l^{|m|}(z) e^{-i m phi}.  ``f`` is (M, C)."""
    f = np.asarray(f, dtype=np.complex128)
    w = np.asarray(weights, dtype=np.float64)
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    C = f.shape[1]
    z = np.clip(pts[:, 2], -1.0, 1.0)
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = np.mod(np.arctan2(pts[:, 1], pts[:, 0]), 2.0 * np.pi)  # favest/core.py:82
    sx, se = seed_table(lt, s)
    wf = w[:, None] * f  # scalar.py:96
    out = np.zeros((flat_size(lt), C), dtype=np.complex128)
    for m in range(lt + 1):
        P = legendre_m(m, lt, z, sx[m], se[m])  # (n_l, M)
        ls = np.arange(m, lt + 1)
        for sgn in ((1,) if m == 0 else (1, -1)):
            mm = sgn * m
            g = np.exp(-1j * mm * phi)[:, None] * wf
            res = P @ g.real + 1j * (P @ g.imag)
            out[ls * ls + ls + mm] = _sigma(mm) * res
    return out


def verify_exactness(points, weights, t):
    """Rule certification (favest/quadrature.py:51-76): the largest
    |sum_i w_i Y(l, m, x_i) - sqrt(4 pi) [l = 0]| over l <= t, 0 <= m <= l, and
    whether it is <= 1e-8.  Real weights: |sum w conj(Y)| = |sum w Y|, so the
    sums are the direct forward of the constant 1."""
    if t < 0:
        raise ValueError(f"certification degree must be non-negative, got {t}")
    n = np.asarray(points).shape[0]
    c = sht_forward_points(np.ones((n, 1)), weights, points, t)[:, 0]
    _, ms = degrees_orders(t)
    sums = c[ms >= 0].copy()
    sums[0] -= np.sqrt(4.0 * np.pi)
    d = float(np.max(np.abs(sums)))
    return d, d <= 1e-8


# --------------------------------------------------------------------------
# Clebsch-Gordan stage — favest/coupling.py:25-78, 143-240; transforms.py:109-180
# --------------------------------------------------------------------------

def _coupling_c(l):
    """favest/coupling.py:25-29 — sqrt((l+1)/(2l+1))."""
    l = np.asarray(l, dtype=np.float64)
    return np.sqrt((l + 1.0) / (2.0 * l + 1.0))


def _coupling_d(l):
    """favest/coupling.py:32-36 — sqrt(l/(2l+1))."""
    l = np.asarray(l, dtype=np.float64)
    return np.sqrt(l / (2.0 * l + 1.0))


def cg_explicit_vec(dl: int, m2: int, l, m) -> np.ndarray:
    """Vectorized favest/coupling.py:39-78 with the same expression order
    (bitwise equal); zero outside |m|<=l, |m-m2|<=l+dl, l+dl>=0, l>=0."""
    l = np.asarray(l, dtype=np.int64)
    m = np.asarray(m, dtype=np.int64)
    j1 = l + dl
    m1 = m - m2
    valid = (l >= 0) & (j1 >= 0) & (np.abs(m) <= l) & (np.abs(m1) <= j1)
    lf = l.astype(np.float64)
    mf = m.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        if dl == -1:
            if m2 == 1:
                v = np.sqrt((l + m) * (lf + mf - 1.0) / ((2.0 * lf) * (2.0 * lf - 1.0)))
            elif m2 == 0:
                v = np.sqrt(((l + m) * (l - m)).astype(np.float64) / (lf * (2.0 * lf - 1.0)))
            else:
                v = np.sqrt((l - m) * (lf - mf - 1.0) / ((2.0 * lf) * (2.0 * lf - 1.0)))
        elif dl == 1:
            if m2 == 1:
                v = np.sqrt((lf - mf + 1.0) * (lf - mf + 2.0) / ((2.0 * lf + 2.0) * (2.0 * lf + 3.0)))
            elif m2 == 0:
                v = -np.sqrt((lf - mf + 1.0) * (lf + mf + 1.0) / ((2.0 * lf + 3.0) * (lf + 1.0)))
            else:
                v = np.sqrt((lf + mf + 1.0) * (lf + mf + 2.0) / ((2.0 * lf + 3.0) * (2.0 * lf + 2.0)))
        else:
            if m2 == 1:
                v = -np.sqrt((l + m) * (lf - mf + 1.0) / (lf * (2.0 * lf + 2.0)))
            elif m2 == 0:
                v = mf / np.sqrt(lf * (lf + 1.0))
            else:
                v = np.sqrt((lf + mf + 1.0) * (l - m) / (lf * (2.0 * lf + 2.0)))
            valid = valid & (l != 0)
    return np.where(valid, v, 0.0)


def cg_tables(lmax: int):
    """favest/coupling.py:143-170 — xi[1..6], mu[1..3] over l <= lmax+1."""
    top = lmax + 1
    ls, ms = degrees_orders(top)
    c1 = _coupling_c(ls + 1)
    dm1 = _coupling_d(np.maximum(ls - 1, 0))
    has = ls >= 1
    xi = {
        1: c1 * cg_explicit_vec(-1, 1, ls + 1, ms + 1),
        2: np.where(has, dm1 * cg_explicit_vec(1, 1, ls - 1, ms + 1), 0.0),
        3: c1 * cg_explicit_vec(-1, -1, ls + 1, ms - 1),
        4: np.where(has, dm1 * cg_explicit_vec(1, -1, ls - 1, ms - 1), 0.0),
        5: c1 * cg_explicit_vec(-1, 0, ls + 1, ms),
        6: np.where(has, dm1 * cg_explicit_vec(1, 0, ls - 1, ms), 0.0),
    }
    mu = {
        1: cg_explicit_vec(0, 1, ls, ms + 1),
        2: cg_explicit_vec(0, 0, ls, ms),
        3: cg_explicit_vec(0, -1, ls, ms - 1),
    }
    return xi, mu


def shift_read(flat, src_lmax, dl, dm, out_lmax):
    """favest/coupling.py:173-184 — flat[(l+dl, m+dm)], zero when out of range.
    ``flat`` may carry trailing axes (the batch)."""
    ls, ms = degrees_orders(out_lmax)
    sl = ls + dl
    sm = ms + dm
    valid = (sl >= 0) & (sl <= src_lmax) & (np.abs(sm) <= sl)
    idx = np.where(valid, sl * sl + sl + sm, 0)
    flat = np.asarray(flat)
    v = valid.reshape(valid.shape + (1,) * (flat.ndim - 1))
    return np.where(v, flat[idx], 0.0).astype(flat.dtype)


def vsht_forward_grid(T, ring_thetas, ring_weights, n_phi, lmax, orders=None):
    """Forward FaVeST on a GL grid (favest/transforms.py:79-147, fast path).

    ``T`` is (N, 3) complex.  Returns (a, b), each (flat_size(lmax),) complex.
    With ``orders`` only the scalar orders needed for those output orders are
    computed (outputs at other orders are then meaningless).
    """
    T = np.asarray(T, dtype=np.complex128)
    t1, t2, t3 = T[:, 0], T[:, 1], T[:, 2]
    combos = np.stack([-t1 + 1j * t2, t1 + 1j * t2, t3], axis=1)  # transforms.py:109-112
    top = lmax + 1
    need = None
    if orders is not None:
        need = set()
        for mo in orders:
            need.update({abs(mo) - 1, abs(mo), abs(mo) + 1})
        need = [x for x in need if 0 <= x <= top]
    f = sht_forward_grid(combos, ring_thetas, ring_weights, n_phi, top, orders=need)
    return cg_forward_assemble(f, lmax)


def vsht_forward_points(T, weights, points, lmax):
    """Forward FaVeST on an arbitrary weighted rule (favest/transforms.py:79-147,
    direct route favest/scalar.py:94-105).  ``T`` is (M, 3) complex."""
    T = np.asarray(T, dtype=np.complex128)
    t1, t2, t3 = T[:, 0], T[:, 1], T[:, 2]
    combos = np.stack([-t1 + 1j * t2, t1 + 1j * t2, t3], axis=1)  # transforms.py:109-112
    f = sht_forward_points(combos, weights, points, lmax + 1)
    return cg_forward_assemble(f, lmax)


def cg_forward_assemble(f, lmax):
    """favest/transforms.py:120-146 — a, b from F^U, F^V, F^W (f is (K_t, 3))."""
    top = lmax + 1
    xi, mu = cg_tables(lmax)
    fu, fv, fw = f[:, 0], f[:, 1], f[:, 2]

    def read(values, dl, dm):
        return shift_read(values, top, dl, dm, lmax)

    a = INV_SQRT2 * (
        read(xi[1] * fu, -1, -1)
        + read(xi[2] * fu, 1, -1)
        + read(xi[3] * fv, -1, 1)
        + read(xi[4] * fv, 1, 1)
    ) + read(xi[5] * fw, -1, 0) + read(xi[6] * fw, 1, 0)
    b = -1j * INV_SQRT2 * (read(mu[1] * fu, 0, -1) + read(mu[3] * fv, 0, 1)) \
        - 1j * read(mu[2] * fw, 0, 0)
    a[0] = 0.0
    b[0] = 0.0
    return a, b


def vsht_adjoint_merged(a, b, lmax):
    """favest/coupling.py:200-240 + favest/transforms.py:165-175: the three
    merged scalar tables (g^X, g^Y, g^Z) of degree lmax+1, shape (K_t, 3)."""
    top = lmax + 1
    xi, mu = cg_tables(lmax)

    def a_at(dl, dm):
        return shift_read(a, lmax, dl, dm, top)

    def b_at(dl, dm):
        return shift_read(b, lmax, dl, dm, top)

    nu1 = a_at(1, 1) * xi[1] - a_at(1, -1) * xi[3]
    nu2 = a_at(-1, 1) * xi[2] - a_at(-1, -1) * xi[4]
    nu3 = 1j * (a_at(1, 1) * xi[1] + a_at(1, -1) * xi[3])
    nu4 = 1j * (a_at(-1, 1) * xi[2] + a_at(-1, -1) * xi[4])
    nu5 = a_at(1, 0) * xi[5]
    nu6 = a_at(-1, 0) * xi[6]
    eta1 = 1j * (b_at(0, 1) * mu[1] - b_at(0, -1) * mu[3])
    eta2 = b_at(0, 1) * mu[1] + b_at(0, -1) * mu[3]
    eta3 = 1j * b_at(0, 0) * mu[2]
    return np.stack(
        [
            -INV_SQRT2 * (nu1 + nu2 + eta1),
            -INV_SQRT2 * (nu3 + nu4 - eta2),
            nu5 + nu6 + eta3,
        ],
        axis=1,
    )


def vsht_adjoint_grid(a, b, lmax, ring_thetas, n_phi, orders=None, spectrum=False):
    """Adjoint FaVeST on a GL grid (favest/transforms.py:150-181, fast path).
    Returns (N, 3) complex Cartesian components, or with ``spectrum`` the ring
    spectra (n_theta, n_phi, 3) of which only the bins of ``orders`` are filled."""
    merged = vsht_adjoint_merged(a, b, lmax)
    return sht_adjoint_grid(merged, lmax + 1, ring_thetas, n_phi, orders=orders, spectrum=spectrum)


def vsht_adjoint_points(a, b, lmax, points):
    """Adjoint FaVeST at scattered points (favest/transforms.py:150-181,
    direct route favest/scalar.py:120-128)."""
    merged = vsht_adjoint_merged(a, b, lmax)
    return sht_adjoint_points(merged, lmax + 1, points)


# --------------------------------------------------------------------------
# seeded generators — SURVEY §8(d), tests/test_transforms.py:22-39
# --------------------------------------------------------------------------

def coef(rng, lmax, law):
    """div then curl table: (N(0,1) + i N(0,1)) * s(l), entry 0 zeroed.
    law 'inv': s = 1/(l(l+1)) (l>=1); 'pow2': s = (1+l)**-2."""
    K = flat_size(lmax)
    ls, _ = degrees_orders(lmax)
    lf = ls.astype(np.float64)
    if law == "inv":
        with np.errstate(divide="ignore"):
            scale = np.where(ls >= 1, 1.0 / np.maximum(lf * (lf + 1.0), 1.0), 0.0)
    elif law == "pow2":
        scale = (1.0 + lf) ** -2
    else:
        raise ValueError(law)
    out = []
    for _ in range(2):
        v = (rng.standard_normal(K) + 1j * rng.standard_normal(K)) * scale
        v[0] = 0.0
        out.append(v)
    return out[0], out[1]


def random_points(rng, n):
    """favest/cli.py:84-88, tests/test_transforms.py:22-24."""
    v = rng.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def tangent_noise(rng, points, sigma):
    """sigma*(N(0,1)+iN(0,1)) per component, projected onto the tangent plane
    (tests/test_transforms.py:27-30)."""
    raw = sigma * (rng.standard_normal(points.shape) + 1j * rng.standard_normal(points.shape))
    raw -= np.sum(raw * points, axis=1)[:, None] * points
    return raw


def rel_l2(x, ref):
    """SURVEY §8(d) parity metric."""
    x = np.asarray(x).ravel()
    ref = np.asarray(ref).ravel()
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (den if den > 0 else 1.0))


def _self_check():  # pragma: no cover - manual
    th, w, nphi = gl_grid(8)
    print(len(th), nphi, math.fsum(w) * nphi)
