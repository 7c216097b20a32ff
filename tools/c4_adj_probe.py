"""C4 adjoint per-call timing (development helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
L = 4096
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=1)
rng = np.random.default_rng(4)
A, Bc = O.coef(rng, L, "pow2")
A = torch.from_numpy(A[None]).cuda(); Bc = torch.from_numpy(Bc[None]).cuda()
T = plan.adjoint(A, Bc); torch.cuda.synchronize()
for rep in range(4):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(); plan.adjoint(A, Bc, T); e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"adj rep {rep}: {e0.elapsed_time(e1):.3f} ms device, host call {1e3*(t1-t0):.3f} ms", flush=True)
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); a, b = plan.forward(T); e1.record(); torch.cuda.synchronize()
    print(f"fwd rep {rep}: {e0.elapsed_time(e1):.3f} ms", flush=True)
