"""CTA-level timeline of the forward Legendre kernel (development helper).
FV_TRACE_CTA=0 python tools/trace_ctas.py"""
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
for _ in range(3): plan.forward(T)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * (4096 * 12))()
lib.fv_debug_trace.argtypes = [ctypes.c_void_p]
lib.fv_debug_trace(ctypes.cast(buf, ctypes.c_void_p))
a = np.frombuffer(buf, dtype=np.int64)[4096 * 8:].reshape(4096, 4)[: L + 2].copy()
t0 = a[:, 0].min(); a[:, :2] -= t0
end = a[:, 1].max()
print("kernel span (ns)", end)
dur = a[:, 1] - a[:, 0]
print("sum CTA durations / (148 * span) = %.3f" % (dur.sum() / (148 * end)))
sms = a[:, 2]
busy = np.zeros(148)
for smid in range(148):
    sel = sms == smid
    busy[smid] = dur[sel].sum()
print("per-SM busy: min %.0f max %.0f mean %.0f ns" % (busy.min(), busy.max(), busy.mean()))
print("first CTA starts: ", sorted(a[:, 0])[:3], " last starts", sorted(a[:, 0])[-3:])
for m in (0, 1, 100, 147, 148, 300, 600, 900, 1025):
    print(f"m={m:5d} start {a[m,0]:8d} end {a[m,1]:8d} dur {dur[m]:7d} sm {sms[m]}")
# idle gaps between consecutive CTAs on the same SM
gaps = []
for smid in range(148):
    ix = np.where(sms == smid)[0]
    st = a[ix, 0]; en = a[ix, 1]; o = np.argsort(st)
    st, en = st[o], en[o]
    gaps += list(st[1:] - en[:-1])
print("inter-CTA gap on an SM: mean %.0f ns, max %.0f" % (np.mean(gaps), np.max(gaps)))
# tail: when does the SM go idle
last_end = np.array([a[sms == s, 1].max() for s in range(148)])
print("SM finish times: min %.0f median %.0f max %.0f" % (last_end.min(), np.median(last_end), last_end.max()))
