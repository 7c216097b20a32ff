"""On-the-fly Legendre forward at a given L, B (development helper for compute-sanitizer)."""
import sys, os
os.environ["FV_PTAB"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
L = int(sys.argv[1]); B = int(sys.argv[2])
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=B)
T = torch.randn(B, len(th) * nphi, 3, dtype=torch.complex128, device="cuda")
fa, fb = plan.forward(T)
torch.cuda.synchronize()
print("ok", L, B, float(fa.abs().sum()))
