"""One forward + adjoint at C2 (L=256, B=16) or C4 (L=4096, B=1) shapes for ncu (development helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
L = int(sys.argv[1]); B = int(sys.argv[2])
th, w, nphi = O.gl_grid(L)
os.environ.setdefault("FV_PTAB", "0")
plan = GridPlan(L, th, w, nphi, max_batch=B)
rng = np.random.default_rng(3)
A = torch.from_numpy(np.stack([O.coef(rng, L, "pow2")[0] for _ in range(B)])).cuda()
Bc = torch.from_numpy(np.stack([O.coef(rng, L, "pow2")[1] for _ in range(B)])).cuda()
T = plan.adjoint(A, Bc)
fa, fb = plan.forward(T)
torch.cuda.synchronize()
print("ok", float(fa.abs().sum()))
