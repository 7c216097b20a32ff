"""`python -m paper_1908_00041_b200 bench` and diagnostics.bench
(favest/cli.py:169-197, favest/diagnostics.py:166-237): same arguments, CSV
header, records and exit codes as the reference's `favest bench`."""

import csv
import math
import subprocess
import sys

import pytest

from gpu_util import cuda_or_skip

HEADER = ["lmax", "n_points", "n_coeffs", "forward_seconds", "adjoint_seconds", "forward_ratio", "adjoint_ratio",
          "threads"]


def _run(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_1908_00041_b200", *args], capture_output=True, text=True,
                          env=env)


def test_cli_usage_errors(tmp_path):
    r = _run()
    assert r.returncode == 2 and "bench" in r.stderr
    r = _run("bench", "--degrees", "0", "--out", str(tmp_path / "b.csv"))
    assert r.returncode == 2 and "bench degrees must be >= 1, got 0" in r.stderr
    r = _run("bench", "--degrees", "4", "--reps", "0", "--out", str(tmp_path / "b.csv"))
    assert r.returncode == 2 and "repetitions must be positive" in r.stderr
    r = _run("bench", "--degrees", "4", "--threads", "0", "--out", str(tmp_path / "b.csv"))
    assert r.returncode == 2 and "thread count must be >= 1" in r.stderr
    import os

    env = dict(os.environ, FAVEST_THREADS="x")
    r = _run("bench", "--degrees", "4", "--out", str(tmp_path / "b.csv"), env=env)
    assert r.returncode == 2 and "FAVEST_THREADS is not an integer" in r.stderr


@pytest.mark.gpu
def test_cli_bench_writes_reference_table(tmp_path):
    cuda_or_skip()
    out = tmp_path / "bench.csv"
    r = _run("bench", "--degrees", "8,16 32", "--reps", "2", "--threads", "3", "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert "wrote 3 bench rows" in r.stdout
    rows = list(csv.reader(open(out, newline="")))
    assert rows[0] == HEADER
    assert [int(x[0]) for x in rows[1:]] == [8, 16, 32]
    for x in rows[1:]:
        L = int(x[0])
        assert int(x[1]) == ((2 * (L + 1) + 2) // 2) * (2 * (L + 1) + 1)
        assert int(x[2]) == L * L + L and int(x[7]) == 3
        assert float(x[3]) > 0 and float(x[4]) > 0
    assert math.isnan(float(rows[1][5])) and rows[1][5] == "nan"


@pytest.mark.gpu
def test_bench_records():
    cuda_or_skip()
    from paper_1908_00041_b200.diagnostics import bench

    recs = bench([4, 12], repetitions=3, seed=5)
    assert [r.lmax for r in recs] == [4, 12]
    assert math.isclose(recs[1].forward_ratio, recs[1].forward_seconds / recs[0].forward_seconds)


def test_error_metrics_matches_reference_definition():
    import numpy as np

    from paper_1908_00041_b200.core import TangentFieldSamples
    from paper_1908_00041_b200.diagnostics import error_metrics

    pts = np.array([[0, 0, 1.0], [1.0, 0, 0], [0, 1.0, 0]])
    a = TangentFieldSamples(pts, np.array([[1, 0, 0], [0, 1j, 0], [0, 0, 2]], dtype=complex))
    b = TangentFieldSamples(pts, a.values + np.array([[0, 1e-3, 0], [0, 0, 0], [0, 0, 0]]))
    w = np.array([1.0, 2.0, 3.0])
    rel, mx = error_metrics(a, b, w)
    assert abs(rel - np.sqrt(1e-6 / (1 + 2 + 12))) <= 1e-18 and mx == 1e-3
    with pytest.raises(ValueError, match="zero norm"):
        error_metrics(TangentFieldSamples(pts, np.zeros((3, 3))), b, w)
