"""C4 Legendre kernel times with the producer or consumer work switched off
(FV_DEBUG_MODE: 1 consumers skip their DMMAs, 2 producers skip the recurrence),
forward and adjoint (development helper; results are meaningless in those modes)."""
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
for name, fn in (("forward", lambda: plan.forward(T, a, b)), ("adjoint", lambda: plan.adjoint(A, Bc, T))):
    fn()
    torch.cuda.synchronize()
    plan.set_profiling(True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = plan.stage_ms()
    plan.set_profiling(False)
    print(f"mode {os.environ.get('FV_DEBUG_MODE', '0')} {name}: legendre {st['legendre'] / 3:.2f} ms", flush=True)
