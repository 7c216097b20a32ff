"""File formats (favest/io.py, favest/quadrature.py:79-139) through the native
codecs of include/favest_io.h, against files and reader outcomes produced by
the reference itself (tests/golden/make_golden.py section 7): writers must be
byte identical, readers bit identical, and malformed input must raise the
reference's exception type and message.  CPU only (no device work)."""

import json
import os

import numpy as np
import pytest

import paper_1908_00041_b200 as fb
from paper_1908_00041_b200 import io as fio

IODIR = os.path.join(os.path.dirname(__file__), "golden", "io")


def _vals():
    return np.load(os.path.join(IODIR, "values.npz"))


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


def _bits_equal(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    both_nan = np.isnan(x) & np.isnan(y)
    return x.shape == y.shape and bool(np.all(both_nan | (x.view(np.uint64) == y.view(np.uint64))))


def test_writers_byte_identical(tmp_path):
    v = _vals()
    L = 12
    c = fb.VectorCoefficients(fb.ScalarCoefficients(L, v["a"]), fb.ScalarCoefficients(L, v["b"]))
    fio.write_coefficients(tmp_path / "c.json", c)
    assert _bytes(tmp_path / "c.json") == _bytes(os.path.join(IODIR, "coef_l12.json"))
    _, rule = fb.gen_gl_tensor(13)
    fio.write_rule_file(tmp_path / "r.rule", rule)
    assert _bytes(tmp_path / "r.rule") == _bytes(os.path.join(IODIR, "gl13.rule"))
    fio.write_samples(tmp_path / "s.csv", fb.TangentFieldSamples(v["points"], v["vals"]))
    assert _bytes(tmp_path / "s.csv") == _bytes(os.path.join(IODIR, "samples_gl13.csv"))
    fio.write_csv(tmp_path / "t.csv", ("l", "err", "name"), [(1, 0.1, "x"), (2, 1e-300, "y")])
    assert _bytes(tmp_path / "t.csv") == _bytes(os.path.join(IODIR, "table.csv"))
    fio.write_csv(tmp_path / "f.csv", ("x", "y"), [(0.1, 2.5), (1e-300, -3.0)])
    assert _bytes(tmp_path / "f.csv") == _bytes(os.path.join(IODIR, "table_f.csv"))


def test_write_csv_header_quoting_and_float32(tmp_path):
    # favest/io.py:136-145 writes the header through csv.writer (quoted when needed) and
    # formats only `float` instances at 17 digits; np.float32 goes through str()
    fio.write_csv(tmp_path / "q.csv", ("a,x", 'q"t'), [(0.1, 1 / 3)])
    assert _bytes(tmp_path / "q.csv") == b'"a,x","q""t"\r\n0.10000000000000001,0.33333333333333331\r\n'
    fio.write_csv(tmp_path / "h.csv", ("a", "b"), [(np.float32(0.1), 1.0), (np.float64(0.2), 2.0)])
    assert _bytes(tmp_path / "h.csv") == b"a,b\r\n0.1,1\r\n0.20000000000000001,2\r\n"


def test_readers_bit_identical():
    v = _vals()
    c = fio.read_coefficients(os.path.join(IODIR, "coef_l12.json"))
    assert c.lmax == 12
    assert _bits_equal(c.div.values.view(np.float64), v["a"].view(np.float64))
    # -0.0 is written "-0", which json.load reads as the int 0: +0.0 in the reference too
    b = v["b"].view(np.float64) + 0.0
    assert _bits_equal(c.curl.values.view(np.float64), b)
    r = fio.read_rule_file(os.path.join(IODIR, "gl13.rule"), 13)
    assert r.kind == "custom" and r.exactness == 13
    assert _bits_equal(r.weights, v["weights"])
    assert np.max(np.abs(r.points - v["points"])) <= 2e-16  # renormalised like the reference
    s = fio.read_samples(os.path.join(IODIR, "samples_gl13.csv"))
    assert np.max(np.abs(s.values - v["vals"])) == 0.0
    assert np.max(np.abs(s.points - v["points"])) <= 1e-15


CASES = json.load(open(os.path.join(IODIR, "cases.json")))


@pytest.mark.parametrize("case", CASES, ids=[f"{c['kind']}-{c['name']}" for c in CASES])
def test_reader_cases_match_reference(tmp_path, case):
    path = str(tmp_path / "case.txt")
    with open(path, "w", newline="") as fh:
        fh.write(case["text"])
    out = case["out"]
    read = {
        "coef": fio.read_coefficients,
        "rule": lambda p: fio.read_rule_file(p, 1),
        "samples": fio.read_samples,
        "design": lambda p: fb.load_design(p, 3),
    }[case["kind"]]
    if not out["ok"]:
        exc = {"ValueError": ValueError, "TypeError": TypeError}[out["type"]]
        with pytest.raises(exc) as info:
            read(path)
        assert type(info.value) is exc
        assert str(info.value).replace(path, "{path}") == out["msg"]
        return
    got = read(path)
    if case["kind"] == "coef":
        assert got.lmax == out["lmax"]
        assert _bits_equal(got.div.values.view(np.float64).reshape(-1, 2), out["a"])
        assert _bits_equal(got.curl.values.view(np.float64).reshape(-1, 2), out["b"])
    elif case["kind"] in ("rule", "design"):
        assert got.kind == out["kind"]
        assert _bits_equal(got.points, out["points"]) and _bits_equal(got.weights, out["weights"])
    else:
        assert _bits_equal(got.points, out["points"])
        vals = np.stack([got.values.real, got.values.imag], axis=-1)
        assert _bits_equal(vals, out["values"])


def test_bundled_icosahedron_certifies_to_five_on_host_geometry():
    r = fb.bundled_design("icosahedron12")
    assert r.kind == "spherical-design" and r.exactness == 5 and len(r.points) == 12
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "exactness.npz"))
    # the reference's own rule, row for row and bit for bit (drop-in: samples built on the
    # reference's bundled_design pass forward_favest's point check and keep their row order)
    assert np.array_equal(r.points, g["ico_points"])
    assert np.array_equal(r.points, np.load(os.path.join(os.path.dirname(__file__), "golden", "direct_ico_l3.npz"))["points"])
    assert np.array_equal(r.weights, np.full(12, 4 * np.pi / 12))
    with pytest.raises(ValueError, match="unknown bundled design"):
        fb.bundled_design("cube")


def test_large_coefficient_file_round_trip(tmp_path):
    """C3 size (L = 1024, 2.1 M complex values): write -> read is lossless."""
    rng = np.random.default_rng(3)
    L = 1024
    K = (L + 1) ** 2
    a = (rng.standard_normal(K) + 1j * rng.standard_normal(K)) * np.exp(rng.uniform(-700, 700, K))
    b = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    a[0] = b[0] = 0
    c = fb.VectorCoefficients(fb.ScalarCoefficients(L, a), fb.ScalarCoefficients(L, b))
    fio.write_coefficients(tmp_path / "big.json", c)
    back = fio.read_coefficients(tmp_path / "big.json")
    assert np.array_equal(back.div.values.view(np.uint64), a.view(np.uint64))
    assert np.array_equal(back.curl.values.view(np.uint64), b.view(np.uint64))
    # the text is valid JSON a plain json.load accepts (spot check the head)
    head = open(tmp_path / "big.json").read(200)
    assert head.startswith('{\n  "L_max": 1024,\n  "a": [[0, 0], [')


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(FileNotFoundError):
        fio.read_coefficients(tmp_path / "nope.json")
    with pytest.raises(FileNotFoundError):
        fio.read_samples(tmp_path / "nope.csv")


def _py_read_columns(text):
    """favest/quadrature.py:112-131 restated (test-local checker for large files)."""
    rows, width = [], None
    for lineno, line in enumerate(text.splitlines(), start=1):
        t = line.split("#", 1)[0].strip()
        if not t:
            continue
        fields = t.replace(",", " ").split()
        if width is None:
            width = len(fields)
        elif len(fields) != width:
            raise ValueError(f"{lineno}: expected {width} columns, got {len(fields)}")
        try:
            rows.append([float(v) for v in fields])
        except ValueError as exc:
            raise ValueError(f"{lineno}: {exc}") from None
    return np.asarray(rows)


@pytest.mark.parametrize("inject", [None, ("width", 150_001), ("float", 199_998), ("float", 3), ("width", 40_000)])
def test_parallel_column_parser_line_numbers(tmp_path, inject):
    """The column parser cuts the text into one chunk per host thread; line
    numbers, widths and the first error must be those of a sequential read."""
    rng = np.random.default_rng(11)
    n = 200_000
    v = rng.standard_normal((n, 3))
    pts = v / np.linalg.norm(v, axis=1, keepdims=True)
    lines = [" ".join(fio.format_float(x) for x in p) for p in pts]
    for k in range(0, n, 997):
        lines[k] = "# comment " + lines[k]
    for k in range(5, n, 1733):
        lines[k] = lines[k] + "   # trailing"
    if inject:
        kind, at = inject
        lines[at - 1] = "0 0" if kind == "width" else "0 0 1e"
    text = "\r\n".join(lines) + "\n"
    path = tmp_path / "big.rule"
    path.write_bytes(text.encode())
    try:
        ref = _py_read_columns(text)
        ref_err = None
    except ValueError as exc:
        ref_err = str(exc)
    if ref_err is None:
        got = fio.read_columns(path)
        assert np.array_equal(got, ref)
    else:
        with pytest.raises(ValueError) as info:
            fio.read_columns(path)
        assert str(info.value) == f"{path}:{ref_err}"
