"""HostPipeline round-trip rate at C3 (L=1024, 4 fields) for several staging depths
(development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import oracle as O
from paper_1908_00041_b200.grid import gl_grid_for
from paper_1908_00041_b200.pipeline import HostPipeline
from paper_1908_00041_b200.plan import GridPlan

L, B = 1024, 4
grid, _ = gl_grid_for(L)
plan = GridPlan.from_grid(grid, L, max_batch=B)
Th = torch.zeros((B, plan.n_points, 3), dtype=torch.complex128, pin_memory=True)
Toh = torch.empty_like(Th, pin_memory=True)
for depth in (2, 3, 4, 6):
    pipe = HostPipeline(plan, depth=depth)
    for _ in range(3):
        pipe.submit_roundtrip(Th, Toh)
    pipe.synchronize()
    n = 30
    q0 = torch.cuda.Event(enable_timing=True)
    q1 = torch.cuda.Event(enable_timing=True)
    q0.record(pipe.h2d)
    for _ in range(n):
        pipe.submit_roundtrip(Th, Toh)
    q1.record(pipe.d2h)
    pipe.synchronize()
    ms = q0.elapsed_time(q1) / n
    print(f"depth {depth}: {ms:.2f} ms per 4-field round trip, {B / ms * 1e3:.0f} fields/s, "
          f"{Th.numel() * 16 / ms / 1e6:.1f} GB/s each way", flush=True)
    del pipe
    torch.cuda.empty_cache()
