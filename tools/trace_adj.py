"""Adjoint Legendre pipeline timeline of one persistent CTA (development helper).
FV_TRACE_CTA=<cta> python tools/trace_adj.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
from paper_1908_00041_b200 import _lib
L, B = 1024, 4
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=B)
a = torch.randn(B, (L + 1) ** 2, dtype=torch.complex128, device="cuda")
b = torch.randn(B, (L + 1) ** 2, dtype=torch.complex128, device="cuda")
plan.adjoint(a, b); torch.cuda.synchronize()
plan.adjoint(a, b); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * (4096 * 12))()
lib.fv_debug_trace.argtypes = [ctypes.c_void_p]
lib.fv_debug_trace(ctypes.cast(buf, ctypes.c_void_p))
raw = np.frombuffer(buf, dtype=np.int64)
t = raw[:4096 * 8].reshape(4096, 8).copy()
ep = raw[4096 * 8:4096 * 12].reshape(4096, 4).copy()
item = t[:, 2] >> 40
t[:, 2] &= (1 << 40) - 1
n = int((t[:, 5] > 0).sum())
t0 = t[:n, 0][t[:n, 0] > 0].min()
t = t[:n] - t0
ep = np.where(ep > 0, ep - t0, 0)
print("stages", n)
print(" sc  item | p_wait p_got p_full | c0_wait c0_got c0_done | c3_wait c3_done | epi")
for s in list(range(0, min(n, 30))) + list(range(max(30, n - 8), n)):
    r = t[s]
    e = ep[s]
    print(f"{s:4d} {int(item[s]):5d} | {r[0]:8d} {r[1]:8d} | {r[3]:8d} {r[4]:8d} {r[5]:8d} | {r[6]:8d} {r[7]:8d} |"
          + (f" epi {e[0]:8d} bar1 +{e[1]-e[0]} bar2 +{e[2]-e[1]} stores +{e[3]-e[2]}" if e[3] else ""))
c0_comp = t[:, 5] - t[:, 4]; c0_idle = t[:, 4] - t[:, 3]
c3_stage = t[:, 7] - t[:, 6]
epi = ep[:n][ep[:n, 3] > 0]
print("consumer0: compute/stage %.0f idle/stage %.0f ; consumer3 stage %.0f" % (c0_comp.mean(), c0_idle.mean(), c3_stage.mean()))
d = np.diff(epi, axis=1)
print("epilogues", len(epi), "avg bar1 %.0f bar2(xch) %.0f stores %.0f" % tuple(d.mean(axis=0)), "total span", t[:, 5].max())
print("sum compute c0", c0_comp.sum(), "sum idle c0", c0_idle.sum(), "sum epi", (epi[:, 3] - epi[:, 0]).sum())
