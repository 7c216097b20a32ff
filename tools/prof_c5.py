"""One C5 scattered adjoint (L=128, M=200,000) for ncu capture (development helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import PointsPlan
L, M = 128, 200_000
rng = np.random.default_rng(5)
v = rng.standard_normal((M, 3)); x = v / np.linalg.norm(v, axis=1, keepdims=True)
a, b = O.coef(rng, L, "inv")
pp = PointsPlan(L)
T = pp.adjoint(torch.from_numpy(x).cuda(), torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda())
torch.cuda.synchronize()
print("ok", float(T.abs().sum()))
