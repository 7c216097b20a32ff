"""adjoint -> forward round trip with scipy's GL rule vs the device rule
(development helper): the round trip is limited by the quadrature weights."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_1908_00041_b200 as fb
from paper_1908_00041_b200.plan import GridPlan

for L in (256, 1024, 4096):
    rng = np.random.default_rng(L)
    a, b = O.coef(rng, L, "pow2")
    A = torch.from_numpy(a[None]).cuda()
    B = torch.from_numpy(b[None]).cuda()
    out = []
    for dev_rule in (False, True):
        grid, _ = fb.gen_gl_tensor(2 * L + 3, on_device=dev_rule)
        plan = GridPlan.from_grid(grid, L)
        T = plan.adjoint(A, B)
        fa, fb_ = plan.forward(T)
        out.append(float(torch.linalg.vector_norm(torch.cat([fa - A, fb_ - B], 1)) /
                         torch.linalg.vector_norm(torch.cat([A, B], 1))))
        plan.close()
        del T
        torch.cuda.empty_cache()
    print(f"L={L}: round trip rel l2 with scipy's rule {out[0]:.2e}, with the device rule {out[1]:.2e}", flush=True)
