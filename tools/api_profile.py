"""Where the public-API time goes at L = 1024 (forward_favest / adjoint_favest
with host numpy arrays): run on the GPU box."""

import time

import numpy as np
import torch

import paper_1908_00041_b200 as fb
from paper_1908_00041_b200 import transforms as tr


def t(label, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label:40s} {1e3 * np.median(ts):8.2f} ms")
    return out


L = 1024
grid, rule = fb.gen_gl_tensor(2 * (L + 1))
rng = np.random.default_rng(0)
vals = rng.standard_normal((len(rule), 3)) + 1j * rng.standard_normal((len(rule), 3))
samples = fb.TangentFieldSamples(rule.points, vals)
K = (L + 1) ** 2
raw = rng.standard_normal((2, K)) + 1j * rng.standard_normal((2, K))
raw[:, 0] = 0
coeffs = fb.VectorCoefficients(fb.ScalarCoefficients(L, raw[0]), fb.ScalarCoefficients(L, raw[1]))
t("forward_favest", lambda: fb.forward_favest(samples, rule, L))
t("adjoint_favest", lambda: fb.adjoint_favest(coeffs, rule))
t("np.allclose points", lambda: np.allclose(samples.points, rule.points, rtol=0.0, atol=1e-12))
t("np.array_equal points", lambda: np.array_equal(samples.points, rule.points))
t("TangentFieldSamples(points, values)", lambda: fb.TangentFieldSamples(rule.points, vals))
t("ascontiguousarray values", lambda: np.ascontiguousarray(vals, dtype=np.complex128))
T = torch.from_numpy(vals).reshape(1, -1, 3)
t("H2D pageable 101 MB", lambda: T.to("cuda"))
Tp = T.pin_memory()
t("H2D pinned 101 MB", lambda: Tp.to("cuda", non_blocking=True))
Td = T.to("cuda")
t("D2H pageable 101 MB", lambda: Td.cpu())
outp = torch.empty_like(T).pin_memory()
t("D2H pinned 101 MB", lambda: outp.copy_(Td, non_blocking=True))
t("numpy copy 101 MB", lambda: vals.copy())
plan = tr.grid_plan(grid, L)
a = torch.from_numpy(raw[0:1].copy()).cuda()
b = torch.from_numpy(raw[1:2].copy()).cuda()
t("plan.forward device", lambda: plan.forward(Td))
t("plan.adjoint device", lambda: plan.adjoint(a, b))
t("grid_plan lookup (hash)", lambda: tr.grid_plan(grid, L))

# pieces of the adjoint's host path (staging.py)
from paper_1908_00041_b200.staging import stager

st = stager(torch.device("cuda", 0))
Tdev = plan.adjoint(a, b)
t("np.empty 101 MB + torch zero_ (first touch)", lambda: torch.from_numpy(np.empty((len(rule), 3), np.complex128)).zero_())
t("stager.to_host 101 MB into fresh pages", lambda: st.to_host(Tdev[0]))
t("stager.to_device coefficients 2 x 16.8 MB", lambda: (st.to_device(raw[0:1]), st.to_device(raw[1:2])))
print("torch threads", torch.get_num_threads())
