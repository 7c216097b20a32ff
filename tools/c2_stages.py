"""C2 (L=256, 16 fields) per-stage device times (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from paper_1908_00041_b200.grid import gl_grid_for
from paper_1908_00041_b200.plan import GridPlan

L, B = 256, 16
grid, _ = gl_grid_for(L)
plan = GridPlan.from_grid(grid, L, max_batch=B)
rng = np.random.default_rng(2)
ab = [O.coef(rng, L, "inv") for _ in range(B)]
a = torch.from_numpy(np.stack([x[0] for x in ab])).cuda()
b = torch.from_numpy(np.stack([x[1] for x in ab])).cuda()
T = plan.adjoint(a, b)
fa, fb = plan.forward(T)
for name, fn in (("forward", lambda: plan.forward(T, fa, fb)), ("adjoint", lambda: plan.adjoint(a, b, T))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    plan.set_profiling(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    st = {k: round(v / 20, 4) for k, v in plan.stage_ms().items()}
    cnt = plan.stage_counts()
    plan.set_profiling(False)
    print(f"{name}: {e0.elapsed_time(e1) / 20:.3f} ms, stages {st}, launches {cnt}", flush=True)
