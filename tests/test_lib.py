"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/favest_b200.h declares, and maps argument errors to the
reference's ValueError messages (validation happens before device work)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1908_00041_b200 import _lib, build

HEADER = os.path.join(build.ROOT, "include", "favest_b200.h")
HEADER_IO = os.path.join(build.ROOT, "include", "favest_io.h")


def header_symbols(path=HEADER):
    txt = open(path).read()
    return sorted(set(re.findall(r"\b(fv_[a-z_]+)\s*\(", txt)))


def test_library_built_and_loads():
    path = build.build()
    assert os.path.exists(path)
    lib = _lib.load()
    assert lib.fv_version().decode().startswith("favest_b200")


def test_exports_every_header_symbol():
    lib = _lib.load()
    assert set(header_symbols(HEADER_IO)) == set(_lib.EXPORTED_IO)
    syms = header_symbols() + header_symbols(HEADER_IO)
    assert set(syms) == set(_lib.EXPORTED) | set(_lib.EXPORTED_IO)
    for s in syms:
        assert hasattr(lib, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", build.LIBPATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", nm), s


def test_sass_is_sm100a_with_dmma():
    out = subprocess.run(["cuobjdump", "-lelf", build.LIBPATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", build.LIBPATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "UBLKCP" in sass or "UTMALDG" in sass  # TMA bulk copies feed the DMMA stages


def _create(L, th, w, nphi, mb=1):
    lib = _lib.load()
    h = ctypes.c_void_p()
    dp = ctypes.POINTER(ctypes.c_double)
    th = np.ascontiguousarray(th, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    rc = lib.fv_plan_create_grid(ctypes.byref(h), L, th.size, nphi, th.ctypes.data_as(dp),
                                 w.ctypes.data_as(dp), mb, 0)
    return rc, lib.fv_last_error().decode()


def test_c_abi_argument_errors_match_reference_messages():
    th = np.linspace(0.3, 2.8, 6)
    w = np.full(6, 0.1)
    rc, msg = _create(0, th, w, 20)
    assert rc == _lib.FV_EINVAL and "lmax >= 1" in msg
    rc, msg = _create(4, th, w, 10)
    assert rc == _lib.FV_EINVAL and msg == "fast-scalar path needs n_phi >= 11 for degree 4, grid has n_phi=10"
    rc, msg = _create(4, th[::-1], w, 20)
    assert rc == _lib.FV_EINVAL and "strictly increasing" in msg
    rc, msg = _create(4, np.array([0.0, 1.0]), w[:2], 20)
    assert rc == _lib.FV_EINVAL and "strictly inside" in msg
    with pytest.raises(ValueError, match="n_phi >= 11"):
        _lib.check(_create(4, th, w, 10)[0])


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="not built"):
        _lib.load(str(tmp_path / "libfavest_b200.so"))
