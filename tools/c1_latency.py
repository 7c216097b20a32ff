"""C1 latency (L=32, one field): eager API calls vs a captured CUDA graph (development helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1908_00041_b200.plan import GridPlan
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
th, w, nphi = O.gl_grid(L)
plan = GridPlan(L, th, w, nphi, max_batch=1)
rng = np.random.default_rng(1)
a0, b0 = O.coef(rng, L, "inv")
A = torch.from_numpy(a0[None]).cuda(); B = torch.from_numpy(b0[None]).cuda()
T = torch.empty((1, len(th) * nphi, 3), dtype=torch.complex128, device="cuda")
a = torch.empty_like(A); b = torch.empty_like(B)
def rt():
    plan.adjoint(A, B, T)
    plan.forward(T, a, b)
for _ in range(5): rt()
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    rt(); torch.cuda.synchronize()
eager = (time.perf_counter() - t0) / n * 1e3
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): rt()
e1.record(); torch.cuda.synchronize()
dev_eager = e0.elapsed_time(e1) / n
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): rt()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    rt()
g.replay(); torch.cuda.synchronize()
ref = np.concatenate([a.cpu().numpy()[0], b.cpu().numpy()[0]])
t0 = time.perf_counter()
for _ in range(n):
    g.replay(); torch.cuda.synchronize()
graph = (time.perf_counter() - t0) / n * 1e3
e0.record()
for _ in range(n): g.replay()
e1.record(); torch.cuda.synchronize()
dev_graph = e0.elapsed_time(e1) / n
ok = O.rel_l2(np.concatenate([a.cpu().numpy()[0], b.cpu().numpy()[0]]), np.concatenate([a0, b0]))
print(f"L={L} adjoint+forward round trip: eager {eager:.3f} ms per call (host-synchronised), {dev_eager:.3f} ms back-to-back; "
      f"CUDA graph {graph:.3f} ms per replay (synchronised), {dev_graph:.3f} ms back-to-back; roundtrip rel {ok:.2e}")
