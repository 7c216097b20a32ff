"""One C4 forward and one C4 adjoint (L=4096, one field) for an ncu capture of the
on-the-fly Legendre kernels (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from paper_1908_00041_b200.plan import GridPlan

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
th, w, nphi = O.gl_grid(L)
rng = np.random.default_rng(4)
A, Bc = O.coef(rng, L, "pow2")
A = torch.from_numpy(A[None]).cuda()
Bc = torch.from_numpy(Bc[None]).cuda()
plan = GridPlan(L, th, w, nphi, max_batch=1)
T = plan.adjoint(A, Bc)
a, b = plan.forward(T)
torch.cuda.synchronize()
print("ok", float((a - A).norm() / A.norm()))
