"""Per-call timing of the staging path pieces (development helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1908_00041_b200.staging import stager

dev = torch.device("cuda", 0)
st = stager(dev)
K = 1025 ** 2
x = (np.random.default_rng(0).standard_normal((1, K)) + 1j).astype(np.complex128)
big = np.random.default_rng(1).standard_normal((2105352, 6)).view(np.complex128)


def t(label, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label:50s} {1e3 * np.median(ts):7.3f} ms (min {1e3 * min(ts):.3f})", flush=True)


t("to_device 16.8 MB", lambda: st.to_device(x))
t("to_device 101 MB", lambda: st.to_device(big))
t("torch .to(dev) 16.8 MB pageable", lambda: torch.from_numpy(x).to(dev))
d = torch.from_numpy(x).to(dev)
t("to_host 16.8 MB (fresh)", lambda: st.to_host(d))
t("torch .cpu() 16.8 MB", lambda: d.cpu())

# the adjoint_favest path at L = 1024, section by section
import paper_1908_00041_b200 as fb
from paper_1908_00041_b200 import transforms as tr

L = 1024
grid, rule = fb.gen_gl_tensor(2 * (L + 1))
rng = np.random.default_rng(0)
raw = rng.standard_normal((2, K)) + 1j * rng.standard_normal((2, K))
raw[:, 0] = 0
coeffs = fb.VectorCoefficients(fb.ScalarCoefficients(L, raw[0]), fb.ScalarCoefficients(L, raw[1]))
for _ in range(2):
    fb.adjoint_favest(coeffs, rule)
for use_pre in (False,):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        points, g2, _ = tr._resolve_grid(rule)
        plan = tr.grid_plan(g2, L)
        res = None
        t1 = time.perf_counter()
        a_d = tr._to_device(np.ascontiguousarray(coeffs.div.values).reshape(1, -1), plan.device)
        b_d = tr._to_device(np.ascontiguousarray(coeffs.curl.values).reshape(1, -1), plan.device)
        t2 = time.perf_counter()
        T = plan.adjoint(a_d, b_d)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        vals = tr._to_host(T[0])
        t4 = time.perf_counter()
        print(f"setup {1e3 * (t1 - t0):.2f} upload {1e3 * (t2 - t1):.2f} device {1e3 * (t3 - t2):.2f} "
              f"download {1e3 * (t4 - t3):.2f} total {1e3 * (t4 - t0):.2f} ms", flush=True)
