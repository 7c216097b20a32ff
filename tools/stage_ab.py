"""A/B helper for kernel variants selected by environment variables (development tool).

    python tools/stage_ab.py L B out.npz      one forward + adjoint on seeded inputs; saves the
                                              results and prints per-stage times (10 timed steps)
    python tools/stage_ab.py --cmp a.npz b.npz   bitwise / relative comparison of two runs

The variants are read by the library once per process, so each configuration
runs in its own process:  FV_CGF_STREAM=1 python tools/stage_ab.py 1024 4 gpurun_out/s1.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    if sys.argv[1] == "--cmp":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        for k in a.files:
            x, y = a[k], b[k]
            same = np.array_equal(x, y)
            rel = float(np.linalg.norm(x - y) / max(np.linalg.norm(x), 1e-300))
            print(f"{k}: bitwise {'EQUAL' if same else 'DIFFERENT'} rel {rel:.3e}")
        return
    import torch

    import oracle as O
    from paper_1908_00041_b200.plan import GridPlan

    L, B, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    th, w, nphi = O.gl_grid(L)
    plan = GridPlan(L, th, w, nphi, max_batch=B)
    rng = np.random.default_rng(3)
    ab = [O.coef(rng, L, "pow2") for _ in range(B)]
    A = torch.from_numpy(np.stack([x[0] for x in ab])).cuda()
    Bc = torch.from_numpy(np.stack([x[1] for x in ab])).cuda()
    T = plan.adjoint(A, Bc)
    fa, fb = plan.forward(T)
    torch.cuda.synchronize()
    np.savez(out, T=T.cpu().numpy(), fa=fa.cpu().numpy(), fb=fb.cpu().numpy())
    for _ in range(3):
        fa, fb = plan.forward(T)
        T2 = plan.adjoint(fa, fb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fa, fb = plan.forward(T)
        T2 = plan.adjoint(fa, fb)
    e1.record()
    torch.cuda.synchronize()
    # per-stage times of the same alternating sequence (stage events; reading them synchronises)
    acc = {}
    plan.set_profiling(True)
    last = plan.stage_ms()
    for _ in range(steps):
        for tag, call in (("f_", lambda: plan.forward(T)), ("a_", lambda: plan.adjoint(fa, fb))):
            call()
            now = plan.stage_ms()
            for k in now:
                acc[tag + k] = acc.get(tag + k, 0.0) + now[k] - last[k]
            last = now
    plan.set_profiling(False)
    cfg = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FV_"))
    print(f"[{cfg or 'default'}] L={L} B={B} step {e0.elapsed_time(e1) / steps:.4f} ms",
          {k: round(v / steps, 4) for k, v in acc.items()})


if __name__ == "__main__":
    main()
