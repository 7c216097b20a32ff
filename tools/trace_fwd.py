"""Forward Legendre pipeline timeline of one CTA (development helper).
FV_TRACE_CTA=<m> python tools/trace_fwd.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
from paper_1908_00041_b200 import _lib
L, B = 1024, 4
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=B)
T = torch.randn(B, len(th) * nphi, 3, dtype=torch.complex128, device="cuda")
plan.forward(T); torch.cuda.synchronize()
plan.forward(T); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * (4096 * 12))()
lib.fv_debug_trace.argtypes = [ctypes.c_void_p]
lib.fv_debug_trace(ctypes.cast(buf, ctypes.c_void_p))
a = np.frombuffer(buf, dtype=np.int64)[:4096 * 8].reshape(4096, 8).copy()
flags = a[:, 2] >> 61
a[:, 2] &= (1 << 61) - 1
n = int((a[:, 3] > 0).sum())
t0 = a[:n, 0][a[:n, 0] > 0].min()
a = a[:n] - t0
print("tiles", n)
print(" t  | prod_wait_start got_empty arrive_full | cons_wait got_full done | flags  | prod_build  cons_compute  cons_idle")
for t in list(range(0, min(n, 40))) + list(range(max(40, n - 10), n)):
    r = a[t]
    print(f"{t:4d} | {r[0]:8d} {r[1]:8d} {r[2]:8d} | {r[3]:8d} {r[4]:8d} {r[5]:8d} | {int(flags[t]):2d} | {r[2]-r[1]:7d} {r[5]-r[4]:7d} {r[4]-r[3]:7d}")
c = a[:n]
print("avg producer build", np.mean(c[:, 2] - c[:, 1]), "avg consumer compute", np.mean(c[:, 5] - c[:, 4]),
      "avg consumer idle", np.mean(c[:, 4] - c[:, 3]), "total", c[:, 5].max())
