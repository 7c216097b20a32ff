#!/usr/bin/env python
"""bench.py — FaVeST forward+adjoint VSHT throughput on B200.

Metric (BASELINE.json): fp64 forward+adjoint VSHT transforms/sec at L=1024,
and the fraction of the FP64 roofline.  One step = forward then adjoint of
every field of the batch (BASELINE configs[2]: L=1024, Gauss-Legendre
1026 x 2052 grid, 4 fields per GPU, coefficients CN(0,1)(1+l)^-2, field =
adjoint(coefficients) + tangent N(0, 1e-3) noise).  value = fields pushed
through forward+adjoint per second over all ranks.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1: one process per GPU.  Under torchrun the ranks come from the
environment (WORLD_SIZE must equal N); without it, bench.py re-launches
itself through ``torch.distributed.run`` with N processes.  Fields are
sharded by batch (weak scaling, no data-path collective); max over ranks of
the CUDA-event time.  Every run also reports, under ``detail``, the C4
workload (L=4096, one field, order-sharded over the N ranks with one NCCL
all-to-all per direction; strong scaling against the single-GPU plan), the
C3 step with the on-the-fly Legendre recurrence (no plan-time tables), and the
C5 scattered adjoint.  --impl reference times the reference algorithm's CPU
implementation (the numpy port in oracle/, spread over all host cores) on
rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 forward+adjoint VSHT transforms/sec at L=1024; fraction of FP64/HBM roofline"
UNIT = "fields/s (forward+adjoint per field)"
# FP64 peaks: DMMA.8x8x4 measured on this pool's B200 (tools/fp64_microbench.cu,
# profiles/r01_fp64_microbench.txt); the datasheet figure is 40 TFLOP/s.
FP64_PEAK_MEASURED = 37.0
FP64_PEAK_DATASHEET = 40.0


def canonical_flops(L: int, B: int) -> dict:
    """SURVEY §8(d) canonical count per direction: folded Legendre contraction
    6*B*n_theta*(L+2)^2 plus three complex ring FFTs 15*B*n_theta*n_phi*log2(n_phi)."""
    nth, nph = L + 2, 2 * L + 4
    leg = 6.0 * B * nth * (L + 2) ** 2
    fft = 15.0 * B * nth * nph * np.log2(nph)
    return {"legendre": leg, "fft": fft, "total": leg + fft}


# DMMA.8x8x4 instructions x 512 flops per C3 launch (ncu sm__inst_executed_pipe_tensor_subpipe_dmma.sum,
# profiles/r02j_legendre_counts.csv; 42.54 M / 41.06 M before the padding pairs and dead chunks were skipped)
EXEC_GFLOP_C3 = {"forward": 39326880 * 512 / 1e9, "adjoint": 39611148 * 512 / 1e9}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """NVML SM clock, max clock and clock-event reasons (the B200_PROFILING.md
    clocks line), read DURING the timed region without touching the launch
    loop: NVML calls take driver locks that stall kernel launches from another
    thread, so all steps are enqueued first and ``drain(event)`` then polls
    every ~2 ms from this thread until the device has executed the timed queue
    (the end event completes)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, torch_device):
        self.dev = torch_device
        self.samples = []
        self.max_mhz = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            # NVML enumerates physical GPUs; map through CUDA_VISIBLE_DEVICES when set
            idx = self.dev.index or 0
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                ids = [x.strip() for x in vis.split(",") if x.strip()]
                if idx < len(ids) and ids[idx].isdigit():
                    idx = int(ids[idx])
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nv, self.h = nv, h
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.ok = True
        except Exception as exc:  # pragma: no cover - NVML missing
            self.err = str(exc)
        return self

    def sample(self):
        """One (SM clock, reasons) reading."""
        if not self.ok:
            return
        nv, h = self.nv, self.h
        try:
            clk = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((float(clk), int(rs)))
        except Exception:
            pass

    def drain(self, end_event):
        """Sample every ~2 ms while the device still runs the enqueued timed steps."""
        while not end_event.query():
            self.sample()
            time.sleep(0.002)

    def __exit__(self, *a):
        pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        reasons = set()
        for _, rs in self.samples:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([c for c, _ in self.samples])), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples), "source": "NVML, 2 ms polling while the device drains the enqueued timed steps"}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_inputs(L: int, B: int, seed: int):
    """BASELINE configs[2] recipe: coefficients first (div then curl per field), then
    tangent noise sigma=1e-3 on top of the adjoint field."""
    import oracle.favest_oracle as O  # only the seeded generators (no oracle compute)

    rng = np.random.default_rng(seed)
    ab = [O.coef(rng, L, "pow2") for _ in range(B)]
    return rng, np.stack([x[0] for x in ab]), np.stack([x[1] for x in ab])


def cpu_port(L: int, n_fields: int, procs: int | None = None):
    """Time the reference algorithm's CPU implementation (the numpy port in
    oracle/, its per-order stage over a pool of one process per host core) on
    ``n_fields`` whole fields of the C3 recipe: forward then adjoint of each,
    nothing sampled or extrapolated.  Returns (fields/s, per-field seconds,
    description, processes)."""
    import oracle.favest_oracle as O
    from oracle.parallel import GridPort

    port = GridPort(L, procs)
    rng, A, Bc = make_inputs(L, 1, seed=3)
    # the C3 field: adjoint of the seeded coefficients + tangent noise (untimed setup)
    T = port.adjoint(A[0], Bc[0]) + O.tangent_noise(rng, O.grid_points(port.th, port.n_phi), 1e-3)
    secs = []
    for _ in range(n_fields):
        t0 = time.perf_counter()
        fa, fb = port.forward(T)
        port.adjoint(fa, fb)
        secs.append(time.perf_counter() - t0)
    desc = (f"numpy port of the reference algorithm (oracle/favest_oracle.py + oracle/parallel.py): one C3 field "
            f"(L={L}, {L + 2}x{2 * L + 4} grid) forward then adjoint in full per timed unit, per-order stage over "
            f"{port.procs} forked processes (BLAS 1 thread each), ring DFTs / CG stages in the parent; "
            f"{n_fields} field(s) timed")
    return 1.0 / float(np.median(secs)), secs, desc, port.procs


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return sum(int(x.get("num_threads", 0)) for x in threadpool_info() if x.get("user_api") == "blas") or None
    except Exception:
        return None


def run_reference(args, rank, world):
    """--impl reference: the path's CPU implementation on the host cores, rank 0 only
    (the reference is pure Python/numpy and cannot travel to the GPU box, so the
    numpy port in oracle/ stands in for it).  Each step is one whole
    C3 field forward then adjoint (a bounded sample of the 4-field C3 step, same
    per-field unit); nothing is extrapolated: value = 1 / median step time."""
    if rank != 0:
        return
    import oracle.favest_oracle as O
    from oracle.parallel import GridPort

    L = args.L
    port = GridPort(L)
    rng, A, Bc = make_inputs(L, 1, seed=3)
    T = port.adjoint(A[0], Bc[0]) + O.tangent_noise(rng, O.grid_points(port.th, port.n_phi), 1e-3)

    def step():
        fa, fb = port.forward(T)
        return port.adjoint(fa, fb)

    for _ in range(args.warmup):
        step()
    secs = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        secs.append(time.perf_counter() - t0)
    wall = time.perf_counter() - t_all
    rate = args.steps / wall
    desc = (f"numpy port of the reference algorithm (oracle/favest_oracle.py + oracle/parallel.py): per step one "
            f"whole C3 field (L={L}, {L + 2}x{2 * L + 4} grid) forward then adjoint, per-order stage over "
            f"{port.procs} forked processes (BLAS 1 thread each), ring DFTs / CG stages in the parent; "
            f"{args.steps} timed steps after {args.warmup} warm-up steps, nothing sampled or extrapolated")
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(L, args.batch, world), "impl": "reference",
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": port.procs, "kind": "port", "sample": desc,
                         "host_cpus": os.cpu_count(), "numpy": np.__version__,
                         "step_s": {"median": float(np.median(secs)), "min": float(min(secs)),
                                    "max": float(max(secs))}, "timed_wall_s": wall},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(L, B, world):
    return {"workload": f"C3 (BASELINE configs[2]): L={L} Gauss-Legendre {L + 2}x{2 * L + 4} grid, "
                        f"{B} fields per GPU, forward then adjoint per step",
            "L": L, "fields_per_gpu": B, "global_batch": B * world, "n_theta": L + 2, "n_phi": 2 * L + 4,
            "parallelism": f"batch-sharded x{world} (no collective)",
            "l2": "inputs exceed the 126 MB L2 (404 MB field batch per GPU), no explicit flush"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # before CUDA is initialised in this process: the port forks its workers
        rate, secs, desc, procs = cpu_port(args.L, args.cpu_fields)
        cpu = {"value": rate, "unit": UNIT, "cores": procs, "kind": "port", "sample": desc,
               "seconds_per_field": secs, "host_cpus": os.cpu_count(), "numpy": np.__version__}
    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        got = dist.get_world_size()
        if got != args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus} but the process group has {got} ranks")
    import oracle.favest_oracle as O
    from paper_1908_00041_b200.grid import gl_grid_for
    from paper_1908_00041_b200.plan import GridPlan

    L, B = args.L, args.batch
    grid, _ = gl_grid_for(L)
    plan = GridPlan.from_grid(grid, L, max_batch=B, device=dev)
    rng, A, Bc = make_inputs(L, B, seed=3 + rank)
    A_d = torch.from_numpy(A).to(dev)
    B_d = torch.from_numpy(Bc).to(dev)
    T0 = plan.adjoint(A_d, B_d)
    pts = torch.from_numpy(O.grid_points(grid.ring_thetas, grid.n_phi)).to(dev)
    # tangent N(0, 1e-3) noise, generated on the device
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    noise = 1e-3 * torch.complex(torch.randn(T0.shape, generator=g, device=dev, dtype=torch.float64),
                                 torch.randn(T0.shape, generator=g, device=dev, dtype=torch.float64))
    noise -= (noise * pts).sum(-1, keepdim=True) * pts
    T = (T0 + noise).contiguous()
    del T0, noise
    a = torch.empty((B, plan.n_coeffs), dtype=torch.complex128, device=dev)
    b = torch.empty_like(a)
    Tout = torch.empty_like(T)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.forward(T, a, b)
        plan.adjoint(a, b, Tout)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    plan.set_profiling(True)  # CUDA events around each stage on the call's stream
    with ClockSampler(dev) as clocks:
        barrier()
        e0.record(stream)
        for i in range(args.steps):
            step()
        e1.record(stream)
        clocks.drain(e1)  # the device is still executing the queued timed steps
        barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    stage_ms = plan.stage_ms()
    stage_n = plan.stage_counts()
    plan.set_profiling(False)
    ms_step = ms_total / args.steps
    value = world * B * args.steps / (ms_total / 1e3)

    # forward-only / adjoint-only device times (separate short loops)
    def timed(fn, n):
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(n):
            fn()
        s1.record(stream)
        barrier()
        return max_over_ranks(s0.elapsed_time(s1)) / n

    n_sub = max(3, args.steps // 2)
    ms_fwd = timed(lambda: plan.forward(T, a, b), n_sub)
    ms_adj = timed(lambda: plan.adjoint(a, b, Tout), n_sub)

    # roofline of the dominant kernel: the Legendre contraction (forward + adjoint launches)
    fl = canonical_flops(L, B)
    n_leg = max(1, stage_n["legendre"])
    leg_ms = stage_ms["legendre"] / n_leg  # average launch (forward and adjoint alternate)
    achieved = fl["legendre"] / (leg_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "legendre_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_MEASURED, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_MEASURED, "traffic": traffic,
                "kernel": "legendre_fwd_kernel / legendre_adj_kernel (FP64 DMMA.8x8x4)",
                "flops_per_launch": fl["legendre"],
                "flops_basis": "6*B*n_theta*(L+2)^2 canonical folded contraction (SURVEY §8(d))",
                "peak_source": "DMMA microbenchmark on this pool (profiles/r01_fp64_microbench.txt); "
                               "datasheet 40 TFLOP/s; MEASURED_PEAKS.json has no FP64 entry",
                "avg_launch_ms": leg_ms, "share_of_step": stage_ms["legendre"] / ms_total}
    if L == 1024 and B == 4:
        # executed DMMA work (the polar skip leaves out whole M-tile k-steps): ncu DMMA
        # instruction counts x 512 flops of the C3 launches, profiles/r02j_legendre_counts.csv
        ex = (EXEC_GFLOP_C3["forward"] + EXEC_GFLOP_C3["adjoint"]) / 2
        roofline["executed_gflop_per_launch"] = dict(EXEC_GFLOP_C3, source="ncu DMMA count x 512")
        roofline["executed_frac"] = ex / (leg_ms / 1e3) / 1e3 / FP64_PEAK_MEASURED
    hbm, hbm_src = hbm_peak()
    step_frac = (2 * fl["total"] / (ms_step / 1e3)) / (FP64_PEAK_DATASHEET * 1e12)

    # end to end: pinned host buffers through the public API, copies inside the timed region.
    # HostPipeline (paper_1908_00041_b200/pipeline.py) overlaps batch k+1's host->device copy,
    # batch k's transforms and batch k-1's device->host copy on three streams (three staging
    # slots: with two, batch k+2's upload waits on batch k's download, which waits on batch
    # k's transforms, so the compute was not hidden); every step's
    # (B, N, 3) samples still cross the link in, and its (B, N, 3) result out.
    e2e = None
    if not args.no_e2e:
        from paper_1908_00041_b200.pipeline import HostPipeline

        Th = torch.empty(T.shape, dtype=T.dtype, pin_memory=True)
        Th.copy_(T)
        Toh = torch.empty_like(Th, pin_memory=True)
        pipe = HostPipeline(plan, depth=3)
        n_e = max(40, args.steps)  # steady state of the streaming pipeline (fill + drain amortised)
        for _ in range(2):
            pipe.submit_roundtrip(Th, Toh)
        pipe.synchronize()
        barrier()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(pipe.h2d)
        for _ in range(n_e):
            pipe.submit_roundtrip(Th, Toh)
        q1.record(pipe.d2h)
        pipe.synchronize()
        barrier()
        ms_e = max_over_ranks(q0.elapsed_time(q1)) / n_e
        # the same API call made one batch at a time (no overlap), for reference
        Td = torch.empty_like(T)

        def serial_step():
            Td.copy_(Th, non_blocking=True)
            plan.forward(Td, a, b)
            plan.adjoint(a, b, Tout)
            Toh.copy_(Tout, non_blocking=True)

        serial_step()
        ms_serial = timed(serial_step, max(2, min(args.steps, 4)))
        bytes_io = T.numel() * 16
        e2e = {"value": world * B / (ms_e / 1e3), "unit": UNIT, "h2d_bytes_per_step": bytes_io,
               "d2h_bytes_per_step": bytes_io, "ms_per_step": ms_e, "steps": n_e,
               "path": "pinned host (B,N,3) -> HostPipeline.submit_roundtrip (GridPlan.forward -> "
                       "GridPlan.adjoint) -> pinned host, copies overlapped across steps",
               "serial_ms_per_step": ms_serial,
               "serial_value": world * B / (ms_serial / 1e3),
               "link_gbs_each_way": bytes_io / (ms_e / 1e3) / 1e9}

    detail_extra = {}
    if not args.no_detail:
        # the same C3 step with the on-the-fly recurrence producer (no plan-time P tables;
        # the mode north_star names and the only one that exists at L=4096)
        detail_extra["on_the_fly"] = on_the_fly_detail(args, world, plan, grid, T, a, b, Tout, timed, dev)
        del plan
        torch.cuda.empty_cache()
        detail_extra["c5"] = c5_detail(args, rank, world, dev, timed)
        detail_extra["c2"] = c2_detail(args, world, dev, timed)
        del T, Tout, a, b
        torch.cuda.empty_cache()
        detail_extra["c4"] = c4_detail(args, rank, world, dev, dist, timed, barrier, max_over_ranks)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(L, B, world),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": int(sum(stage_n.values())),
            "detail": {
                "forward_ms": ms_fwd, "adjoint_ms": ms_adj,
                "forward_fields_per_s": world * B / (ms_fwd / 1e3),
                "adjoint_fields_per_s": world * B / (ms_adj / 1e3),
                "stage_ms_per_step": {k: v / args.steps for k, v in stage_ms.items()},
                "canonical_gflop_per_direction": fl["total"] / 1e9,
                "step_fraction_of_fp64_roofline_datasheet": step_frac,
                "forward_fraction_of_roofline": (fl["total"] / (ms_fwd / 1e3)) / (FP64_PEAK_DATASHEET * 1e12),
                "adjoint_fraction_of_roofline": (fl["total"] / (ms_adj / 1e3)) / (FP64_PEAK_DATASHEET * 1e12),
                "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
                "polar_skip_threshold": "2^-100 (values below are exact zeros; SURVEY §7 hard part 2)",
                "launches_note": "our kernels in the timed region, counted by the plan's stage marks: per step "
                                 "and 4-field group fft_fold (forward FFT + fold), legendre_fwd, cg_fwd_tile, "
                                 "cg_adj_tile, legendre_adj, ring_fft2 (inverse)",
                **detail_extra,
            },
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# detail entries of the headline line
# ---------------------------------------------------------------------------
def on_the_fly_detail(args, world, plan, grid, T, a, b, Tout, timed, dev):
    """The C3 step on a plan built with FV_PTAB=0: the Legendre producers run the
    block-rescaled three-term recurrence beside the DMMAs instead of streaming
    plan-time tables (north_star's on-the-fly recurrence)."""
    from paper_1908_00041_b200.plan import GridPlan

    L, B = args.L, args.batch
    old = os.environ.get("FV_PTAB")
    os.environ["FV_PTAB"] = "0"
    try:
        p2 = GridPlan.from_grid(grid, L, max_batch=B, device=dev)
    finally:
        if old is None:
            del os.environ["FV_PTAB"]
        else:
            os.environ["FV_PTAB"] = old

    def step():
        p2.forward(T, a, b)
        p2.adjoint(a, b, Tout)

    for _ in range(3):
        step()
    n = max(5, args.steps // 2)
    p2.set_profiling(True)
    ms = timed(step, n)
    st, cnt = p2.stage_ms(), p2.stage_counts()
    p2.set_profiling(False)
    # bitwise-independent check: the on-the-fly forward matches the table-mode forward
    a2, b2 = p2.forward(T)
    a1, b1 = plan.forward(T)
    import torch

    rel = float(torch.linalg.vector_norm(torch.cat([a2 - a1, b2 - b1])) / torch.linalg.vector_norm(torch.cat([a1, b1])))
    p2.close()
    fl = canonical_flops(L, B)
    leg_ms = st["legendre"] / max(1, cnt["legendre"])
    return {"ms_per_step": ms, "value": world * B / (ms / 1e3),
            "unit": UNIT, "steps": n,
            "legendre_avg_launch_ms": leg_ms,
            "legendre_frac_of_measured_dmma_peak": fl["legendre"] / (leg_ms / 1e3) / 1e12 / FP64_PEAK_MEASURED,
            "stage_ms_per_step": {k: v / n for k, v in st.items()},
            "step_fraction_of_fp64_roofline_datasheet": (2 * fl["total"] / (ms / 1e3)) / (FP64_PEAK_DATASHEET * 1e12),
            "forward_rel_l2_vs_table_mode": rel,
            "note": "plan built with FV_PTAB=0: P-bar by the on-the-fly recurrence, no plan-time tables"}


def c2_detail(args, world, dev, timed):
    """BASELINE configs[1]: L=256, a batch of 16 fields per GPU (default_rng(2), the
    1/(l(l+1)) law), forward and adjoint each timed separately."""
    import torch

    import oracle.favest_oracle as O  # seeded generators only
    from paper_1908_00041_b200.grid import gl_grid_for
    from paper_1908_00041_b200.plan import GridPlan

    L2, B2 = 256, 16
    grid, _ = gl_grid_for(L2)
    plan = GridPlan.from_grid(grid, L2, max_batch=B2, device=dev)
    rng = np.random.default_rng(2)
    ab = [O.coef(rng, L2, "inv") for _ in range(B2)]
    a = torch.from_numpy(np.stack([x[0] for x in ab])).to(dev)
    b = torch.from_numpy(np.stack([x[1] for x in ab])).to(dev)
    T = plan.adjoint(a, b)
    fa, fb = plan.forward(T)
    for _ in range(3):
        plan.adjoint(a, b, T)
        plan.forward(T, fa, fb)
    n = 20
    ms_a = timed(lambda: plan.adjoint(a, b, T), n)
    ms_f = timed(lambda: plan.forward(T, fa, fb), n)
    rt = float(torch.linalg.vector_norm(torch.cat([fa - a, fb - b], 1)) / torch.linalg.vector_norm(torch.cat([a, b], 1)))
    plan.close()
    fl = canonical_flops(L2, B2)
    frac = lambda ms: fl["total"] / (ms / 1e3) / (FP64_PEAK_DATASHEET * 1e12)  # noqa: E731
    return {"workload": "C2 (BASELINE configs[1]): L=256 Gauss-Legendre 258x516 grid, 16 fields per GPU, forward and "
                        "adjoint timed separately", "forward_ms": ms_f, "adjoint_ms": ms_a,
            "forward_fields_per_s": world * B2 / (ms_f / 1e3), "adjoint_fields_per_s": world * B2 / (ms_a / 1e3),
            "forward_fraction_of_fp64_roofline_datasheet": frac(ms_f),
            "adjoint_fraction_of_fp64_roofline_datasheet": frac(ms_a),
            "roundtrip_rel_l2": rt}


def c5_detail(args, rank, world, dev, timed):
    """BASELINE configs[4]: adjoint of one L=128 field at M=200,000 scattered points
    (default_rng(5): points, then coefficients with the 1/(l(l+1)) law); points
    sharded across the ranks (no exchange), coefficients replicated."""
    import torch

    import oracle.favest_oracle as O  # seeded generators only
    from paper_1908_00041_b200.plan import PointsPlan

    L5, M = 128, 200_000
    rng = np.random.default_rng(5)
    pts = O.random_points(rng, M)
    a, b = O.coef(rng, L5, "inv")
    lo, hi = rank * M // world, (rank + 1) * M // world
    pp = PointsPlan(L5, max_batch=1, device=dev)
    xyz = torch.from_numpy(np.ascontiguousarray(pts[lo:hi])).to(dev)
    a_d = torch.from_numpy(a[None]).to(dev)
    b_d = torch.from_numpy(b[None]).to(dev)
    Tp = pp.adjoint(xyz, a_d, b_d)
    for _ in range(3):
        pp.adjoint(xyz, a_d, b_d, Tp)
    n = 20
    ms = timed(lambda: pp.adjoint(xyz, a_d, b_d, Tp), n)
    # parity guard: 64 points of this rank's shard against the oracle
    sel = np.linspace(0, hi - lo - 1, 64).astype(int)
    ref = O.vsht_adjoint_points(a, b, L5, pts[lo:hi][sel])
    rel = O.rel_l2(Tp[0].cpu().numpy()[sel], ref)
    pp.close()
    gflop = 47.37  # 40.56 contraction + 6.81 recurrence
    return {"workload": "C5 (BASELINE configs[4]): adjoint at M=200,000 scattered points, L=128, one field, "
                        f"points sharded x{world}",
            "ms_per_transform": ms, "transforms_per_s": 1e3 / ms, "points_per_s": M / (ms / 1e3),
            "canonical_gflop": gflop, "fraction_of_fp64_roofline_datasheet": gflop / (ms / 1e3) / 1e3 / FP64_PEAK_DATASHEET,
            "frac_of_measured_dmma_peak": gflop / (ms / 1e3) / 1e3 / FP64_PEAK_MEASURED,
            "scaling": "strong", "rel_l2_vs_oracle_64_points": rel}


def c4_detail(args, rank, world, dev, dist, timed, barrier, max_over_ranks):
    """BASELINE configs[3]: one L=4096 field (4098 x 8196 grid), forward then adjoint
    per step.  N > 1: order-sharded over the ranks (dist.py: ring-sharded field,
    m-sharded contraction, one NCCL all-to-all per direction).  Rank 0 also times
    the single-GPU plan on the same field (the strong-scaling reference)."""
    import torch

    import oracle.favest_oracle as O  # seeded generators only
    from paper_1908_00041_b200.grid import gl_grid_for
    from paper_1908_00041_b200.plan import GridPlan

    L4 = 4096
    grid, _ = gl_grid_for(L4)
    rng = np.random.default_rng(4)
    A, Bc = O.coef(rng, L4, "pow2")
    a_full = torch.from_numpy(A[None]).to(dev)
    b_full = torch.from_numpy(Bc[None]).to(dev)
    n = args.c4_steps
    fl = canonical_flops(L4, 1)
    out = {"workload": "C4 (BASELINE configs[3]): L=4096 Gauss-Legendre 4098x8196 grid, one field, forward then "
                       "adjoint per step", "steps": n, "canonical_gflop_per_direction": fl["total"] / 1e9}
    if world > 1:
        from paper_1908_00041_b200.dist import make_plan

        sp = make_plan(L4, grid, 1, rank, world, dev)
        T_local = sp.adjoint(a_full, b_full)
        a = torch.zeros_like(a_full)
        b = torch.zeros_like(b_full)
        Tout = torch.empty_like(T_local)

        def step():
            sp.forward(T_local, a, b)
            sp.adjoint(a, b, Tout)

        for _ in range(2):
            step()
        ms = timed(step, n)
        rel = float(torch.linalg.vector_norm(Tout - T_local) / torch.linalg.vector_norm(T_local))
        out.update({"sharded_ms_per_step": ms, "parallelism": f"order-sharded x{world} (NCCL all-to-all per direction)",
                    "rank0_rings": list(sp.me.rings), "rank0_orders": list(sp.me.orders),
                    "roundtrip_rel_l2": max_over_ranks(rel),
                    "sharded_fraction_of_fp64_roofline_datasheet":
                        (2 * fl["total"] / (ms / 1e3)) / (FP64_PEAK_DATASHEET * 1e12 * world)})
        del sp, T_local, Tout, a, b
        torch.cuda.empty_cache()
    barrier()
    if rank == 0:
        plan = GridPlan.from_grid(grid, L4, max_batch=1, device=dev)
        T = plan.adjoint(a_full, b_full)
        a = torch.empty_like(a_full)
        b = torch.empty_like(b_full)
        Tout = torch.empty_like(T)

        def step1():
            plan.forward(T, a, b)
            plan.adjoint(a, b, Tout)

        for _ in range(2):
            step1()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream(dev)
        torch.cuda.synchronize(dev)
        s0.record(st)
        for _ in range(n):
            step1()
        s1.record(st)
        torch.cuda.synchronize(dev)
        ms1 = s0.elapsed_time(s1) / n
        rel1 = float(torch.linalg.vector_norm(Tout - T) / torch.linalg.vector_norm(T))
        out.update({"single_gpu_ms_per_step": ms1, "single_gpu_roundtrip_rel_l2": rel1,
                    "single_gpu_fraction_of_fp64_roofline_datasheet":
                        (2 * fl["total"] / (ms1 / 1e3)) / (FP64_PEAK_DATASHEET * 1e12)})
        if world > 1:
            out["speedup_vs_single_gpu"] = ms1 / out["sharded_ms_per_step"]
        if world == 1 and not args.no_rank_share:
            # the order-sharded step's per-rank device work at 2 / 4 / 8 ranks, each simulated
            # rank timed alone on this GPU (tools/c4_rank_share.py; no kernel waits on another
            # rank), plus the all-to-all volume at NVLink speed (modelled, not measured)
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from c4_rank_share import rank_share

            del Tout
            rs = rank_share(plan, T, a_full, b_full, worlds=(2, 4, 8), single=ms1)
            out["order_sharded_projection"] = {
                "method": "per-rank device work of dist.OrderShardedPlan (make_plan defaults: one chunk, cost-balanced orders) timed "
                          "rank by rank on one GPU, transposes replaced by local copies; NVLink time = max bytes "
                          "sent per rank / 900 GB/s (modelled: one GPU)",
                **{str(w): {"slowest_rank_ms": v["slowest_rank_ms"], "nvlink_ms_at_900GBs": v["nvlink_ms_at_900GBs"],
                            "speedup_compute_only": v["speedup_vs_single_gpu_plan_compute_only"],
                            "speedup_with_serial_nvlink": v["speedup_vs_single_gpu_plan_with_serial_nvlink"]}
                   for w, v in rs["ranks"].items()}}
        plan.close()
        del T, a, b
        torch.cuda.empty_cache()
    barrier()
    return out


# ---------------------------------------------------------------------------
# C4: one L=4096 field, order-sharded over the ranks (strong scaling)
# ---------------------------------------------------------------------------
def run_c4(args, rank, world, local_rank):
    """BASELINE configs[3]: L=4096, one field, forward + adjoint per step, order-sharded
    across the N ranks (paper_1908_00041_b200/dist.py: ring-sharded field, m-sharded
    contraction, one NCCL all-to-all per direction)."""
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    dist.init_process_group("nccl", device_id=dev)
    import oracle.favest_oracle as O
    from paper_1908_00041_b200.dist import make_plan
    from paper_1908_00041_b200.grid import gl_grid_for

    L = args.L if args.L != 1024 else 4096
    grid, _ = gl_grid_for(L)
    sp = make_plan(L, grid, 1, rank, world, dev)
    rng = np.random.default_rng(4)
    A, Bc = O.coef(rng, L, "pow2")
    a_full = torch.from_numpy(A[None]).to(dev)
    b_full = torch.from_numpy(Bc[None]).to(dev)
    T_local = sp.adjoint(a_full, b_full)  # this rank's rings of adjoint(coefficients)
    a = torch.zeros_like(a_full)
    b = torch.zeros_like(b_full)
    Tout = torch.empty_like(T_local)

    def step():
        sp.forward(T_local, a, b)
        sp.adjoint(a, b, Tout)

    def barrier():
        dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        barrier()
        e0.record(stream)
        for i in range(args.steps):
            step()
        e1.record(stream)
        clocks.drain(e1)  # the device is still executing the queued timed steps
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    # parity guard on the timed outputs: adjoint(forward(adjoint(c))) vs adjoint(c) on this rank's rings
    rel = float(torch.linalg.vector_norm(Tout - T_local) / torch.linalg.vector_norm(T_local))
    rel = max_over_ranks(rel)
    fl = canonical_flops(L, 1)
    if rank == 0:
        lay = sp.me
        line = {
            "metric": "fp64 forward+adjoint VSHT pairs/sec at L=4096 (order-sharded)",
            "value": 1.0 / (ms / 1e3), "unit": "fields/s (forward+adjoint per field)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C4 (BASELINE configs[3]): L=4096 Gauss-Legendre 4098x8196 grid, one field, "
                                   "forward then adjoint per step, order-sharded", "L": L, "global_batch": 1,
                       "parallelism": f"order-sharded x{world} (NCCL all-to-all per direction)",
                       "rank0_rings": list(lay.rings), "rank0_orders": list(lay.orders)},
            "clocks": clocks.summary(),
            "detail": {"canonical_gflop_per_direction": fl["total"] / 1e9,
                       "fraction_of_fp64_roofline_datasheet": (2 * fl["total"] / (ms / 1e3)) / (FP64_PEAK_DATASHEET * 1e12),
                       "roundtrip_rel_l2": rel},
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def dry_run(args, rank, world):
    """--dry-run: the multi-rank plumbing of run_ours (process group, world check,
    barrier, max over ranks, rank 0 prints one line) over gloo on the CPU."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
        if dist.get_world_size() != args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus} but the process group has {dist.get_world_size()} ranks")
        dist.barrier()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "dry_run": True, "max_over_ranks": float(t.item()),
                          "config": workload_config(args.L, args.batch, world)}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch(n: int):
    """``--gpus N`` without a torchrun environment: re-execute this script under
    ``torch.distributed.run`` with N processes on this node (127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--L", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=4, help="fields per GPU")
    ap.add_argument("--cpu-fields", type=int, default=3, help="whole fields timed for cpu_baseline")
    ap.add_argument("--c4-steps", type=int, default=5, help="timed steps of the C4 detail entry")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-detail", action="store_true", help="skip the on-the-fly / C5 / C4 detail entries")
    ap.add_argument("--no-rank-share", action="store_true", help="skip the C4 per-rank projection at N=1")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: the same re-launch and rank set-up over gloo, "
                         "one max-over-ranks reduction, the JSON line's rank bookkeeping (no timing)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c4"],
                    help="c3: batch-sharded L=1024 (the headline); c4: one L=4096 field, order-sharded")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args.gpus)  # does not return
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    if world > 1:
        # communicator set-up lines (ranks, NVLink/NVLS transport) on stderr, stdout keeps the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.dry_run:
        dry_run(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "c4":
        run_c4(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
