"""File formats of the reference (favest/io.py), with the formatting and
parsing done by the native codecs of ``include/favest_io.h``.

Same names, signatures, file bytes and error behaviour as ``favest/io.py``:
every float is written with 17 significant digits (a lossless double round
trip), readers accept '#' comment lines and blank lines, malformed content
raises ``ValueError`` naming the file.  Python opens, reads and writes the
files (so missing files raise the same ``OSError``s); the C++ side turns
whole tables into text on all host threads and parses text back into
float64 arrays (at L = 1024 a coefficient file is 2.1 M complex values,
~80 MB of text).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .core import (
    QuadratureRule,
    ScalarCoefficients,
    TangentFieldSamples,
    VectorCoefficients,
    from_spherical,
    to_spherical,
)

SAMPLES_HEADER = ("theta", "phi", "t1_re", "t1_im", "t2_re", "t2_im", "t3_re", "t3_im")


def format_float(x: float) -> str:
    """favest/io.py:30-31"""
    return format(float(x), ".17g")


def _take(lib, ptr, n) -> bytes:
    try:
        return ctypes.string_at(ptr, n) if n else b""
    finally:
        lib.fv_io_free(ptr)


def _table_text(data: np.ndarray, sep: str, crlf: bool) -> bytes:
    lib = _lib.load()
    d = np.ascontiguousarray(data, dtype=np.float64)
    nrows, ncols = (d.shape[0], d.shape[1]) if d.ndim == 2 else (0, 1)
    out, n = ctypes.c_void_p(), ctypes.c_longlong(0)
    _lib.check(lib.fv_io_format_table(d.ctypes.data if d.size else None, nrows, ncols, ord(sep), int(crlf),
                                      ctypes.byref(out), ctypes.byref(n)))
    return _take(lib, out.value, n.value)


def _read_bytes(path) -> bytes:
    with open(path, "rb") as fh:
        return fh.read()


def read_columns(path) -> np.ndarray:
    """favest/quadrature.py:112-131 (``_read_columns``): whitespace/comma
    separated numeric columns, '#' comments, constant width."""
    lib = _lib.load()
    text = _read_bytes(path)
    data, nr, nc = ctypes.c_void_p(), ctypes.c_longlong(0), ctypes.c_int(0)
    _lib.check(lib.fv_io_parse_columns(text, len(text), 0, ctypes.byref(data), ctypes.byref(nr), ctypes.byref(nc)),
               path)
    try:
        arr = np.ctypeslib.as_array(ctypes.cast(data.value, ctypes.POINTER(ctypes.c_double)),
                                    shape=(nr.value * nc.value,)).copy()
    finally:
        lib.fv_io_free(data.value)
    return arr.reshape(nr.value, nc.value)


def renormalize(points: np.ndarray, path) -> np.ndarray:
    """favest/quadrature.py:134-139"""
    from .core import check_unit

    norms = np.sqrt(np.sum(points * points, axis=1))
    err = float(np.max(np.abs(norms - 1.0)))
    if err > 1e-6:
        raise ValueError(f"points in {path} deviate from the unit sphere by {err:.3e} (> 1e-6)")
    return check_unit(points / norms[:, None])


def write_rule_file(path, rule: QuadratureRule) -> None:
    """Write a 4-column "x y z w" rule file (favest/io.py:33-38)."""
    pts = np.asarray(rule.points, dtype=np.float64)
    head = f"# quadrature rule: {len(pts)} points, exactness {rule.exactness}, kind {rule.kind}\n"
    body = _table_text(np.column_stack([pts, np.asarray(rule.weights, dtype=np.float64)]), " ", False)
    with open(path, "wb") as fh:
        fh.write(head.encode())
        fh.write(body)


def read_rule_file(path, exactness: int, kind: str | None = None) -> QuadratureRule:
    """Read "x y z" (equal weights) or "x y z w" rule files (favest/io.py:41-59)."""
    data = read_columns(path)
    if data.shape[1] not in (3, 4):
        raise ValueError(f"{path}: rule files have 3 or 4 columns, got {data.shape[1]}")
    points = renormalize(data[:, :3], path)
    if data.shape[1] == 3:
        n = len(points)
        weights = np.full(n, 4.0 * np.pi / n)
        return QuadratureRule(points, weights, exactness, kind or "spherical-design")
    return QuadratureRule(points, data[:, 3].copy(), exactness, kind or "custom")


def write_coefficients(path, coeffs: VectorCoefficients) -> None:
    """{"L_max": L, "a": [[re, im], ...], "b": ...} (favest/io.py:62-77)."""
    lib = _lib.load()
    a = np.ascontiguousarray(coeffs.div.values, dtype=np.complex128)
    b = np.ascontiguousarray(coeffs.curl.values, dtype=np.complex128)
    out, n = ctypes.c_void_p(), ctypes.c_longlong(0)
    _lib.check(lib.fv_io_format_coefficients(int(coeffs.lmax), a.ctypes.data, b.ctypes.data, ctypes.byref(out),
                                             ctypes.byref(n)))
    text = _take(lib, out.value, n.value)
    with open(path, "wb") as fh:
        fh.write(text)


def read_coefficients(path) -> VectorCoefficients:
    """favest/io.py:80-95"""
    lib = _lib.load()
    text = _read_bytes(path)
    lmax, pa, pb = ctypes.c_int(0), ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(lib.fv_io_parse_coefficients(text, len(text), ctypes.byref(lmax), ctypes.byref(pa), ctypes.byref(pb)),
               path)
    size = (lmax.value + 1) ** 2
    out = []
    try:
        for p in (pa.value, pb.value):
            arr = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(2 * size,))
            out.append(ScalarCoefficients(lmax.value, arr.copy().view(np.complex128)))
    finally:
        lib.fv_io_free(pa.value)
        lib.fv_io_free(pb.value)
    return VectorCoefficients(out[0], out[1])


def write_samples(path, samples: TangentFieldSamples) -> None:
    """CSV theta, phi, t1_re ... t3_im (favest/io.py:98-108)."""
    thetas, phis = to_spherical(samples.points)
    values = np.asarray(samples.values, dtype=np.complex128)
    table = np.empty((len(thetas), 8))
    table[:, 0], table[:, 1] = thetas, phis
    table[:, 2::2], table[:, 3::2] = values.real, values.imag
    with open(path, "wb") as fh:
        fh.write((",".join(SAMPLES_HEADER) + "\r\n").encode())
        fh.write(_table_text(table, ",", True))


def read_samples(path) -> TangentFieldSamples:
    """favest/io.py:111-133"""
    lib = _lib.load()
    text = _read_bytes(path)
    data, nr, nc = ctypes.c_void_p(), ctypes.c_longlong(0), ctypes.c_int(0)
    _lib.check(lib.fv_io_parse_columns(text, len(text), 1, ctypes.byref(data), ctypes.byref(nr), ctypes.byref(nc)),
               path)
    try:
        arr = np.ctypeslib.as_array(ctypes.cast(data.value, ctypes.POINTER(ctypes.c_double)),
                                    shape=(nr.value * 8,)).copy().reshape(nr.value, 8)
    finally:
        lib.fv_io_free(data.value)
    points = from_spherical(arr[:, 0], arr[:, 1])
    values = arr[:, 2::2] + 1j * arr[:, 3::2]
    return TangentFieldSamples(points, values)


def write_csv(path, header, rows) -> None:
    """CSV table with floats at 17 significant digits (favest/io.py:136-145);
    all-float tables go through the native formatter, mixed rows through csv."""
    import csv
    import io as _io

    rows = list(rows)
    # the native formatter only for values the reference formats itself (isinstance
    # float: Python floats and np.float64, not np.float32, which csv writes as str())
    if rows and all(isinstance(v, float) for r in rows for v in r) and len({len(r) for r in rows}) == 1:
        head = _io.StringIO(newline="")
        csv.writer(head).writerow(header)  # csv quoting of header fields, as the reference
        with open(path, "wb") as fh:
            fh.write(head.getvalue().encode())
            fh.write(_table_text(np.asarray(rows, dtype=np.float64), ",", True))
        return

    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(header)
        for row in rows:
            writer.writerow(format_float(v) if isinstance(v, float) else v for v in row)


__all__ = [
    "SAMPLES_HEADER", "format_float", "write_rule_file", "read_rule_file", "write_coefficients",
    "read_coefficients", "write_samples", "read_samples", "write_csv", "read_columns",
]
