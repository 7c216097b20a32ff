"""C5 scattered adjoint (L=128, M=200,000) device time (development helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import PointsPlan
L, M = 128, 200_000
rng = np.random.default_rng(5)
v = rng.standard_normal((M, 3)); x = v / np.linalg.norm(v, axis=1, keepdims=True)
a, b = O.coef(rng, L, "inv")
pp = PointsPlan(L)
xd, ad, bd = torch.from_numpy(x).cuda(), torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda()
T = pp.adjoint(xd, ad, bd)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    T = pp.adjoint(xd, ad, bd)
e1.record(); torch.cuda.synchronize()
ref = O.vsht_adjoint_points(a, b, L, x[:64])
print(f"C5 adjoint {e0.elapsed_time(e1) / 10:.3f} ms, rel l2 vs oracle (64 points) {O.rel_l2(T[0, :64].cpu().numpy(), ref):.2e}")
