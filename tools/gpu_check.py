"""Quick GPU sanity / parity / timing check (development helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan, PointsPlan

def c1():
    g = np.load("tests/golden/roundtrip_l32.npz")
    L = 32
    plan = GridPlan(L, g["ring_thetas"], g["ring_weights"], int(g["n_phi"]), max_batch=2)
    a = torch.from_numpy(g["a"]).reshape(1, -1).cuda(); b = torch.from_numpy(g["b"]).reshape(1, -1).cuda()
    T = plan.adjoint(a, b); torch.cuda.synchronize()
    print("C1 adj rel", O.rel_l2(T[0].cpu().numpy(), g["T"]), flush=True)
    fa, fb = plan.forward(torch.from_numpy(g["T"]).reshape(1, -1, 3).cuda()); torch.cuda.synchronize()
    print("C1 fwd rel", O.rel_l2(np.concatenate([fa[0].cpu().numpy(), fb[0].cpu().numpy()]), np.concatenate([g["fa"], g["fb"]])), flush=True)
    fa, fb = plan.forward(torch.from_numpy(g["Tn"]).reshape(1, -1, 3).cuda()); torch.cuda.synchronize()
    print("C1 fwd noisy rel", O.rel_l2(np.concatenate([fa[0].cpu().numpy(), fb[0].cpu().numpy()]), np.concatenate([g["fna"], g["fnb"]])), flush=True)
    for f in ("scattered_l16_m300", "scattered_l9_m64"):
        s = np.load(f"tests/golden/{f}.npz")
        pp = PointsPlan(int(s["lmax"]))
        T = pp.adjoint(torch.from_numpy(s["points"]).cuda(), torch.from_numpy(s["a"]).reshape(1,-1).cuda(), torch.from_numpy(s["b"]).reshape(1,-1).cuda())
        print(f, "rel", O.rel_l2(T[0].cpu().numpy(), s["T"]), flush=True)

def batch_check(L, B, seed):
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(seed)
    A = []; Bc = []
    for _ in range(B):
        a, b = O.coef(rng, L, "inv"); A.append(a); Bc.append(b)
    A = np.stack(A); Bc = np.stack(Bc)
    plan = GridPlan(L, th, w, nphi, max_batch=B)
    T = plan.adjoint(torch.from_numpy(A).cuda(), torch.from_numpy(Bc).cuda())
    Tn = T.cpu().numpy()
    fa, fb = plan.forward(T); fa = fa.cpu().numpy(); fb = fb.cpu().numpy()
    for bi in (0, B - 1):
        Tr = O.vsht_adjoint_grid(A[bi], Bc[bi], L, th, nphi)
        ra, rb = O.vsht_forward_grid(Tn[bi], th, w, nphi, L)
        print(f"L={L} B={B} field {bi}: adj rel {O.rel_l2(Tn[bi], Tr):.3e} fwd rel {O.rel_l2(np.concatenate([fa[bi], fb[bi]]), np.concatenate([ra, rb])):.3e} roundtrip {O.rel_l2(np.concatenate([fa[bi], fb[bi]]), np.concatenate([A[bi], Bc[bi]])):.3e}", flush=True)

def timing(L, B, reps=10):
    th, w, nphi = O.gl_grid(L)
    plan = GridPlan(L, th, w, nphi, max_batch=B)
    rng = np.random.default_rng(3)
    A = torch.from_numpy(np.stack([O.coef(rng, L, "pow2")[0] for _ in range(B)])).cuda()
    Bc = torch.from_numpy(np.stack([O.coef(rng, L, "pow2")[1] for _ in range(B)])).cuda()
    T = plan.adjoint(A, Bc)
    plan.forward(T); torch.cuda.synchronize()
    for name, fn in (("fwd", lambda: plan.forward(T)), ("adj", lambda: plan.adjoint(A, Bc))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        plan.set_profiling(True); fn(); st = plan.stage_ms(); plan.set_profiling(False)
        Kt = (L + 2) ** 2; nth = L + 2
        flops = 6 * B * nth * Kt + 15 * B * nth * nphi * np.log2(nphi)
        print(f"L={L} B={B} {name}: {ms:.3f} ms  {flops/ms/1e9:.2f} TF/s canonical  stages {st}", flush=True)

if __name__ == "__main__":
    what = sys.argv[1:] or ["c1", "b64", "t"]
    if "c1" in what: c1()
    if "b64" in what:
        batch_check(64, 3, 7); batch_check(40, 5, 8)
    if "b256" in what: batch_check(256, 4, 2)
    if "t" in what:
        timing(256, 16); timing(1024, 4)

def c4_timing(reps=3):
    L = 4096
    th, w, nphi = O.gl_grid(L)
    t0 = time.time()
    plan = GridPlan(L, th, w, nphi, max_batch=1)
    torch.cuda.synchronize()
    print("C4 plan", time.time() - t0, "s", flush=True)
    rng = np.random.default_rng(4)
    A, Bc = O.coef(rng, L, "pow2")
    A = torch.from_numpy(A[None]).cuda(); Bc = torch.from_numpy(Bc[None]).cuda()
    T = plan.adjoint(A, Bc); plan.forward(T); torch.cuda.synchronize()
    plan.set_profiling(True)
    for name, fn in (("fwd", lambda: plan.forward(T)), ("adj", lambda: plan.adjoint(A, Bc))):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        before = plan.stage_ms()
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        after = plan.stage_ms()
        st = {k: (after[k] - before[k]) / reps for k in after}
        print(f"C4 L=4096 B=1 {name}: {ms:.3f} ms  stages {st}", flush=True)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "c4":
    c4_timing()

def c5_timing(reps=5, B=1):
    """C5: adjoint at M = 200,000 scattered points, L = 128 (B fields)."""
    L, M = 128, 200_000
    rng = np.random.default_rng(5)
    v = rng.standard_normal((M, 3)); x = v / np.linalg.norm(v, axis=1, keepdims=True)
    cs = [O.coef(rng, L, "inv") for _ in range(B)]
    a = np.stack([c[0] for c in cs]); b = np.stack([c[1] for c in cs])
    pp = PointsPlan(L, max_batch=B)
    X = torch.from_numpy(x).cuda(); A = torch.from_numpy(a).cuda(); Bc = torch.from_numpy(b).cuda()
    T = pp.adjoint(X, A, Bc); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): pp.adjoint(X, A, Bc)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    Kt = (L + 2) ** 2
    flops = B * 24 * ((L + 2) * (L + 3) // 2) * M + 4 * ((L + 2) * (L + 3) // 2) * M
    print(f"C5 L={L} M={M} B={B}: {ms:.3f} ms  {B*1e3/ms:.1f} transforms/s  {flops/ms/1e9:.2f} TF/s (SURVEY canonical 47.37 GFLOP per field)", flush=True)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "c5":
    c5_timing()
    c5_timing(B=4)

def c5f_timing(reps=5):
    """Direct-route forward at C5 shapes: M = 200,000 weighted scattered points, L = 128."""
    L, M = 128, 200_000
    rng = np.random.default_rng(5)
    x = O.random_points(rng, M)
    w = np.full(M, 4 * np.pi / M)
    for B in (1, 4):
        T = np.stack([O.tangent_noise(rng, x, 1.0) for _ in range(B)])
        pp = PointsPlan(L, max_batch=B)
        X = torch.from_numpy(x).cuda(); W = torch.from_numpy(w).cuda(); Td = torch.from_numpy(T).cuda()
        pp.forward(X, W, Td); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): pp.forward(X, W, Td)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        flops = B * 24 * ((L + 2) * (L + 3) // 2) * M + 4 * ((L + 2) * (L + 3) // 2) * M
        print(f"C5-forward L={L} M={M} B={B}: {ms:.3f} ms  {B*1e3/ms:.1f} transforms/s  {flops/ms/1e9:.2f} TF/s canonical", flush=True)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "c5f":
    c5f_timing()
