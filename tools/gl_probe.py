"""Device Gauss-Legendre rule vs scipy (development helper): weight differences by
position and exactness defects (float64 Legendre recurrence)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy.special import roots_legendre

from paper_1908_00041_b200.grid import gauss_legendre_device


def defect(x, w, n):
    p0, p1 = np.ones(n), x.copy()
    d = max(abs(np.dot(w, p0) - 2.0), abs(np.dot(w, p1)))
    for l in range(2, 2 * n):
        p0, p1 = p1, ((2 * l - 1) * x * p1 - (l - 1) * p0) / l
        d = max(d, abs(np.dot(w, p1)))
    return d


for n in (34, 130, 515, 1026, 2050, 4098):
    th, w = gauss_legendre_device(n)
    x, gw = roots_legendre(n)
    x, gw = x[::-1], gw[::-1]
    rel = np.abs(w / gw - 1)
    print(f"n={n}: |dx| max {np.max(np.abs(np.cos(th) - x)):.1e}; weight rel diff pole {rel[0]:.1e} "
          f"first 1% {np.max(rel[:max(1, n // 100)]):.1e} middle {np.max(rel[n // 4:n - n // 4]):.1e}; "
          f"exactness defect device {defect(np.cos(th), w, n):.1e} scipy {defect(x, gw, n):.1e}", flush=True)
