"""Per-rank device time of the order-sharded C4 step, measured on one GPU.

Only one B200 is reachable from this build, so the 2/4/8-GPU run cannot be
timed end to end.  What can be measured without making kernels wait on one
another: every simulated rank's own work (its ring DFTs, the packing of its
sends, the Legendre / CG of its order chunks, its synthesis, its inverse ring
DFTs), timed rank by rank with CUDA events on one device, with the transposes
replaced by local copies (dist.simulate_* bookkeeping).  The step time of an
N-GPU run is then bounded below by the slowest rank's work and above by that
plus the all-to-all volume at NVLink speed (reported separately, not measured).

    python tools/c4_rank_share.py [L] [chunks] [cost|degrees]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from paper_1908_00041_b200.dist import CudaStages, OrderShardedPlan, _unflatten
from paper_1908_00041_b200.plan import GridPlan

def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rank_share(base, T, A, Bc, worlds=(1, 2, 4, 8), chunks=1, balance="cost", single=None, stages_detail=False):
    """Per-rank forward / adjoint device times of the order-sharded step on ``base``'s
    grid for each world size (one field: T (1, N, 3), A / Bc (1, K)); see module doc."""
    L, nth, nphi = base.lmax, base.n_theta, base.n_phi
    if single is None:
        a0, b0 = base.forward(T)
        single = timed(lambda: (base.forward(T, a0, b0), base.adjoint(A, Bc, T)))
    out = {"L": L, "chunks": chunks, "balance": balance, "single_gpu_plan_ms_per_step": single, "ranks": {}}
    stages = CudaStages(base)
    cost = base.order_cost() if balance == "cost" else None
    for world in worlds:
        plans = [OrderShardedPlan(stages, L, nth, nphi, 1, r, world, base.device, chunks=chunks, cost=cost)
                 for r in range(world)]
        T4 = T.view(1, nth, nphi, 3)
        Tl = [T4[:, p.me.rings[0]:p.me.rings[1]].reshape(1, -1, 3).contiguous() for p in plans]
        # every rank's sends (computed once; each receiving rank reuses them)
        S = [p.forward_fft(t).clone() for p, t in zip(plans, Tl)]
        sends = [[_unflatten(p.forward_send(s, q)) for q in range(chunks)] for p, s in zip(plans, S)]
        a = torch.zeros_like(A)
        b = torch.zeros_like(Bc)
        adj_sends = [[_unflatten(p.adjoint_send(A, Bc, q)) for q in range(chunks)] for p in plans]
        # each rank's receive buffers (the blocks of every source in rank order)
        recv_f = [[torch.cat([sends[g][q][h].reshape(-1) for g in range(world)]) for q in range(chunks)]
                  for h in range(world)]
        recv_a = [[torch.cat([adj_sends[g][q][h].reshape(-1) for g in range(world)]) for q in range(chunks)]
                  for h in range(world)]
        per = []
        vol = 0
        for h, p in enumerate(plans):
            def fwd():
                s = p.forward_fft(Tl[h])
                for q in range(chunks):
                    p.forward_send(s, q)
                    p.forward_finish(recv_f[h][q], 1, a, b, q)

            def adj():
                for q in range(chunks):
                    p.adjoint_send(A, Bc, q)
                    p.adjoint_unpack(recv_a[h][q], 1, q)
                p.adjoint_finish(1, Tl[h])

            rec = {"rank": h, "rings": list(p.me.rings), "orders": list(p.me.orders)}
            for name, fn in (("forward", fwd), ("adjoint", adj)):
                base.set_profiling(stages_detail)
                rec[name + "_ms"] = timed(fn)
                if stages_detail:
                    rec[name + "_stage_ms"] = {k: v / 4 for k, v in base.stage_ms().items()}
                base.set_profiling(False)
            rec["step_ms"] = rec["forward_ms"] + rec["adjoint_ms"]
            # bytes this rank sends to other ranks per step (forward + adjoint transposes)
            sent = sum(int(x.numel()) * 16 for q in range(chunks) for g, x in enumerate(sends[h][q]) if g != h)
            sent += sum(int(x.numel()) * 16 for q in range(chunks) for g, x in enumerate(adj_sends[h][q]) if g != h)
            rec["sent_bytes"] = sent
            vol = max(vol, sent)
            per.append(rec)
        slow = max(x["step_ms"] for x in per)
        out["ranks"][world] = {"per_rank": per, "slowest_rank_ms": slow,
                               "max_bytes_sent_per_rank": vol,
                               "nvlink_ms_at_900GBs": vol / 900e9 * 1e3,
                               "speedup_vs_single_gpu_plan_compute_only": single / slow,
                               "speedup_vs_single_gpu_plan_with_serial_nvlink": single / (slow + vol / 900e9 * 1e3)}
        del plans, S, sends, adj_sends, recv_f, recv_a
        torch.cuda.empty_cache()
    return out


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    balance = sys.argv[3] if len(sys.argv) > 3 else "cost"
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(4)
    A, Bc = O.coef(rng, L, "pow2")
    A = torch.from_numpy(A[None]).cuda()
    Bc = torch.from_numpy(Bc[None]).cuda()
    base = GridPlan(L, th, w, nphi, max_batch=1)
    T = base.adjoint(A, Bc)
    torch.cuda.synchronize()
    out = rank_share(base, T, A, Bc, chunks=chunks, balance=balance, stages_detail=True)
    for world, v in out["ranks"].items():
        print(f"world {world}: slowest rank {v['slowest_rank_ms']:.2f} ms, sends "
              f"{v['max_bytes_sent_per_rank'] / 1e6:.0f} MB ({v['nvlink_ms_at_900GBs']:.2f} ms at 900 GB/s); "
              f"single-GPU plan {out['single_gpu_plan_ms_per_step']:.2f} ms -> "
              f"x{v['speedup_vs_single_gpu_plan_compute_only']:.2f} (compute only), "
              f"x{v['speedup_vs_single_gpu_plan_with_serial_nvlink']:.2f} (+ serial NVLink)", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
