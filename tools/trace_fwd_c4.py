"""Single-field (C4) forward Legendre pipeline timeline of one CTA (development
helper): FV_TRACE_CTA=<order> python tools/trace_fwd_c4.py [L]

The consumer columns need a library built with -DFV_TRACE_CONSUMERS (the stamps
cost ~1 ms of the 22.9 ms forward, so they are not in the default build)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from paper_1908_00041_b200 import _lib
from paper_1908_00041_b200.plan import GridPlan

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=1)
T = torch.randn(1, len(th) * nphi, 3, dtype=torch.complex128, device="cuda")
plan.forward(T)
torch.cuda.synchronize()
plan.forward(T)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * (4096 * 12))()
lib.fv_debug_trace.argtypes = [ctypes.c_void_p]
lib.fv_debug_trace(ctypes.cast(buf, ctypes.c_void_p))
a = np.frombuffer(buf, dtype=np.int64)[:4096 * 8].reshape(4096, 8).copy()
a[:, 2] &= (1 << 61) - 1
n = int((a[:, 5] > 0).sum())
t0 = a[:n, 0][a[:n, 0] > 0].min()
c = a[:n, :6] - t0
print("tiles", n, "(first 4096 of the CTA)")
print("   t | prod: wait  got_empty  arrived | cons: wait  got_full  issued | build  cons_idle  cons_step")
for t in list(range(0, 24)) + list(range(max(24, n - 8), n)):
    r = c[t]
    step = c[t, 5] - c[t - 1, 5] if t else 0
    print(f"{t:4d} | {r[0]:9d} {r[1]:9d} {r[2]:9d} | {r[3]:9d} {r[4]:9d} {r[5]:9d} | {r[2]-r[1]:6d} {r[4]-r[3]:6d} {step:6d}")
steps = np.diff(c[:, 5])
idle = c[:, 4] - c[:, 3]
build = c[:, 2] - c[:, 1]
wait_empty = c[:, 1] - c[:, 0]
print(f"per tile (cycles): consumer step median {np.median(steps):.0f} mean {steps.mean():.0f}; consumer wait on full "
      f"median {np.median(idle):.0f} mean {idle.mean():.0f}; producer build median {np.median(build):.0f}; producer "
      f"wait on empty median {np.median(wait_empty):.0f}; producer lead (arrive before consumer wait) median "
      f"{np.median(c[:, 3] - c[:, 2]):.0f}")
