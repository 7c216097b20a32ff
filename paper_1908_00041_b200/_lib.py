"""ctypes binding of ``libfavest_b200.so`` (C ABI: include/favest_b200.h).

The library is the only compute path: if it is missing or cannot be loaded
the calls raise — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

from .build import LIBPATH

FV_OK, FV_EINVAL, FV_ECUDA, FV_ENCCL, FV_ENOMEM, FV_ETYPE = 0, 1, 2, 3, 4, 6

#: every symbol include/favest_b200.h declares
EXPORTED = (
    "fv_version", "fv_last_error", "fv_plan_create_grid", "fv_plan_create_points",
    "fv_plan_destroy", "fv_plan_info", "fv_forward_grid", "fv_adjoint_grid",
    "fv_adjoint_points", "fv_forward_points", "fv_set_profiling", "fv_stage_ms", "fv_stage_count",
    "fv_ring_fft", "fv_forward_orders", "fv_adjoint_orders", "fv_order_cost",
    "fv_forward_orders_packed", "fv_adjoint_orders_packed", "fv_gauss_legendre",
    "fv_forward_scalar_grid", "fv_adjoint_scalar_grid", "fv_forward_scalar_points", "fv_adjoint_scalar_points",
)

#: every symbol include/favest_io.h declares (host-only file codecs)
EXPORTED_IO = (
    "fv_io_free", "fv_io_format_table", "fv_io_format_coefficients", "fv_io_parse_columns",
    "fv_io_parse_coefficients",
)

_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and prototype the shared library."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIBPATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{os.path.basename(p)} is not built; run `python -m paper_1908_00041_b200.build` "
            "(the CUDA extension is the only compute path, there is no CPU fallback)"
        )
    lib = ctypes.CDLL(p)
    vp, i, d, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    sig = {
        "fv_version": (ctypes.c_char_p, []),
        "fv_last_error": (ctypes.c_char_p, []),
        "fv_plan_create_grid": (i, [ctypes.POINTER(vp), i, i, i, dp, dp, i, i]),
        "fv_plan_create_points": (i, [ctypes.POINTER(vp), i, i, i]),
        "fv_plan_destroy": (None, [vp]),
        "fv_plan_info": (i, [vp, ip, ip, ip, ip, ip]),
        "fv_forward_grid": (i, [vp, vp, vp, vp, i, vp]),
        "fv_adjoint_grid": (i, [vp, vp, vp, vp, i, vp]),
        "fv_adjoint_points": (i, [vp, vp, ll, vp, vp, vp, i, vp]),
        "fv_forward_points": (i, [vp, vp, vp, ll, vp, vp, vp, i, vp]),
        "fv_set_profiling": (i, [vp, i]),
        "fv_stage_ms": (d, [vp, i]),
        "fv_stage_count": (i, [vp, i]),
        "fv_ring_fft": (i, [vp, i, vp, ll, ll, ll, vp, ll, ll, ll, i, vp]),
        "fv_forward_orders": (i, [vp, vp, ll, ll, ll, i, i, vp, vp, i, i, i, i, i, vp]),
        "fv_adjoint_orders": (i, [vp, vp, vp, i, i, i, vp, ll, ll, ll, i, i, vp]),
        "fv_order_cost": (i, [vp, dp]),
        "fv_gauss_legendre": (i, [i, dp, dp, i]),
        "fv_forward_orders_packed": (i, [vp, vp, vp, ll, i, i, vp, vp, i, i, i, i, i, vp]),
        "fv_adjoint_orders_packed": (i, [vp, vp, vp, i, i, i, vp, vp, ll, i, i, vp]),
        "fv_forward_scalar_grid": (i, [vp, vp, vp, i, i, vp]),
        "fv_adjoint_scalar_grid": (i, [vp, vp, vp, i, i, vp]),
        "fv_forward_scalar_points": (i, [vp, vp, vp, ll, vp, vp, i, i, vp]),
        "fv_adjoint_scalar_points": (i, [vp, vp, ll, vp, vp, i, i, vp]),
        "fv_io_free": (None, [vp]),
        "fv_io_format_table": (i, [vp, ll, i, i, i, ctypes.POINTER(vp), ctypes.POINTER(ll)]),
        "fv_io_format_coefficients": (i, [i, vp, vp, ctypes.POINTER(vp), ctypes.POINTER(ll)]),
        "fv_io_parse_columns": (i, [ctypes.c_char_p, ll, i, ctypes.POINTER(vp), ctypes.POINTER(ll), ip]),
        "fv_io_parse_coefficients": (i, [ctypes.c_char_p, ll, ip, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int, path=None) -> None:
    """Map a C status code to the reference's exception types ("{path}" in a
    file codec's message becomes the file name)."""
    if rc == FV_OK:
        return
    msg = load().fv_last_error().decode() or f"favest_b200 error {rc}"
    if path is not None:
        msg = msg.replace("{path}", str(path))
    if rc == FV_EINVAL:
        raise ValueError(msg)
    if rc == FV_ETYPE:
        raise TypeError(msg)
    if rc == FV_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
