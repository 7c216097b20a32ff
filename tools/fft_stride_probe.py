"""Inverse ring DFT (two-ring kernel) with the field's interleaved output vs a contiguous one (development helper)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
L, B = 1024, 4
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=B)
nr = B * len(th)
S = torch.randn(3, nr, nphi, dtype=torch.complex128, device="cuda")   # ring-major input (contiguous rings)
T = torch.empty(nr * nphi * 3, dtype=torch.complex128, device="cuda")
lib = plan.lib
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def run(inv, in_strides, out_strides, reps=10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(2): lib.fv_ring_fft(plan._h, inv, S.data_ptr(), *in_strides, T.data_ptr(), *out_strides, nr, s)
    e0.record()
    for _ in range(reps): lib.fv_ring_fft(plan._h, inv, S.data_ptr(), *in_strides, T.data_ptr(), *out_strides, nr, s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
n = nphi
print("inverse, ring-major in -> (B,N,3) out:", run(1, (nr * n, n, 1), (1, 3 * n, 3)))
print("inverse, ring-major in -> contiguous rings out:", run(1, (nr * n, n, 1), (nr * n, n, 1)))
print("forward, (B,N,3) in -> contiguous out:", run(0, (1, 3 * n, 3), (nr * n, n, 1)))
print("forward, contiguous in -> contiguous out:", run(0, (nr * n, n, 1), (nr * n, n, 1)))
