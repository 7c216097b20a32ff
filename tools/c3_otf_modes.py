"""C3 (L=1024, 4 fields) Legendre kernel times on the on-the-fly producer (FV_PTAB=0)
and table mode, with FV_DEBUG_MODE isolation (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from paper_1908_00041_b200.plan import GridPlan

L, B = 1024, 4
th, w, nphi = O.gl_grid(L)
rng = np.random.default_rng(3)
ab = [O.coef(rng, L, "pow2") for _ in range(B)]
A = torch.from_numpy(np.stack([x[0] for x in ab])).cuda()
Bc = torch.from_numpy(np.stack([x[1] for x in ab])).cuda()
plan = GridPlan(L, th, w, nphi, max_batch=B)
T = plan.adjoint(A, Bc)
a, b = plan.forward(T)
torch.cuda.synchronize()
for name, fn in (("forward", lambda: plan.forward(T, a, b)), ("adjoint", lambda: plan.adjoint(A, Bc, T))):
    fn()
    torch.cuda.synchronize()
    plan.set_profiling(True)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    st = plan.stage_ms()
    plan.set_profiling(False)
    print(f"ptab {os.environ.get('FV_PTAB', '1')} mode {os.environ.get('FV_DEBUG_MODE', '0')} {name}: "
          f"legendre {st['legendre'] / 5:.3f} ms", flush=True)
