"""Time the file codecs against the reference's own writers / readers at the
C3 sizes (L = 1024: coefficient file of 2 x 1,050,625 complex values; the
2,105,352-point GL grid's sample CSV and rule file).  Host-only; run in the
build container, where /root/reference is importable:

    python tools/io_bench.py [--skip-reference]
"""

import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1908_00041_b200 as fb  # noqa: E402
from paper_1908_00041_b200 import io as fio  # noqa: E402


def timed(fn, reps=1):
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    skip_ref = "--skip-reference" in sys.argv
    L = 1024
    K = (L + 1) ** 2
    rng = np.random.default_rng(3)
    a = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    b = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    a[0] = b[0] = 0
    grid, rule = fb.gen_gl_tensor(2 * L + 3)
    pts = rule.points
    vals = rng.standard_normal((len(pts), 3)) + 1j * rng.standard_normal((len(pts), 3))
    d = tempfile.mkdtemp()
    ours = {
        "write_coefficients": lambda: fio.write_coefficients(
            d + "/m.json", fb.VectorCoefficients(fb.ScalarCoefficients(L, a), fb.ScalarCoefficients(L, b))),
        "read_coefficients": lambda: fio.read_coefficients(d + "/m.json"),
        "write_samples": lambda: fio.write_samples(d + "/m.csv", fb.TangentFieldSamples(pts, vals)),
        "read_samples": lambda: fio.read_samples(d + "/m.csv"),
        "write_rule_file": lambda: fio.write_rule_file(d + "/m.rule", rule),
        "read_rule_file": lambda: fio.read_rule_file(d + "/m.rule", 2 * L + 3),
    }
    res = {k: timed(f, 3) for k, f in ours.items()}
    sizes = {"coefficients": os.path.getsize(d + "/m.json"), "samples": os.path.getsize(d + "/m.csv"),
             "rule": os.path.getsize(d + "/m.rule")}
    ref = {}
    if not skip_ref:
        sys.path.insert(0, "/root/reference/pkg/src")
        from favest import core as rc, io as rio
        from favest.quadrature import gen_gl_tensor as rgl

        _, rrule = rgl(2 * L + 3)
        rv = rc.VectorCoefficients(rc.ScalarCoefficients(L, a), rc.ScalarCoefficients(L, b))
        refs = {
            "write_coefficients": lambda: rio.write_coefficients(d + "/r.json", rv),
            "read_coefficients": lambda: rio.read_coefficients(d + "/r.json"),
            "write_samples": lambda: rio.write_samples(d + "/r.csv", rc.TangentFieldSamples(pts, vals)),
            "read_samples": lambda: rio.read_samples(d + "/r.csv"),
            "write_rule_file": lambda: rio.write_rule_file(d + "/r.rule", rrule),
            "read_rule_file": lambda: rio.read_rule_file(d + "/r.rule", 2 * L + 3),
        }
        ref = {k: timed(f) for k, f in refs.items()}
        for x in ("json", "csv", "rule"):
            same = open(d + f"/m.{x}", "rb").read() == open(d + f"/r.{x}", "rb").read()
            print(f"{x}: byte identical = {same}")
    print(f"host threads {os.cpu_count()}; sizes {sizes}")
    print("| call | this library (s) | reference (s) | speed-up |")
    print("|---|---|---|---|")
    for k, v in res.items():
        r = ref.get(k)
        print(f"| {k} | {v:.3f} | {r:.2f} | {r / v:.0f}x |" if r else f"| {k} | {v:.3f} | - | - |")


if __name__ == "__main__":
    main()
