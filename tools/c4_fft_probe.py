"""C4 (L=4096, one field) per-stage device times of the forward and the adjoint
(development helper): ring DFT (+ fused fold), Legendre, Clebsch-Gordan, for the
default ring DFT and FV_FFT=rp (cuFFT sub-DFTs + combine)."""
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
ref = None
for mode in ("", "rp"):
    if mode:
        os.environ["FV_FFT"] = mode
    plan = GridPlan(L, th, w, nphi, max_batch=1)
    os.environ.pop("FV_FFT", None)
    T = plan.adjoint(A, Bc)
    a, b = plan.forward(T)
    torch.cuda.synchronize()
    if ref is None:
        ref = (T.clone(), a.clone())
    else:
        print(f"  vs default: adjoint rel {float((T - ref[0]).norm() / ref[0].norm()):.2e}, "
              f"forward rel {float((a - ref[1]).norm() / ref[1].norm()):.2e}")
    for name, fn in (("forward", lambda: plan.forward(T, a, b)), ("adjoint", lambda: plan.adjoint(A, Bc, T))):
        fn()
        torch.cuda.synchronize()
        plan.set_profiling(True)
        n = 5
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        st = {k: v / n for k, v in plan.stage_ms().items()}
        plan.set_profiling(False)
        print(f"[{mode or 'default'}] {name}: {e0.elapsed_time(e1) / n:.3f} ms  stages " +
              " ".join(f"{k} {v:.3f}" for k, v in st.items()), flush=True)
    rt = float(torch.cat([a - A, b - Bc], 1).norm() / torch.cat([A, Bc], 1).norm())
    print(f"[{mode or 'default'}] roundtrip rel {rt:.2e}")
    plan.close()
    del plan, T, a, b
    torch.cuda.empty_cache()
