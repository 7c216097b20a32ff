"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the numpy oracle, on the BASELINE configs' seeded inputs.

Tolerance: relative l2 <= 1e-11 in float64 (BASELINE.json north_star);
observed values are 1e-16..1e-13.
"""

import os

import numpy as np
import pytest

import oracle as O
from gpu_util import cuda_or_skip

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(autouse=True)
def _need_cuda():
    cuda_or_skip()


def _plan(L, th, w, nphi, B=1):
    from paper_1908_00041_b200.plan import GridPlan

    return GridPlan(L, th, w, nphi, max_batch=B)


def _t(x):
    torch = cuda_or_skip()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("lmax", [8, 17, 32])
def test_golden_roundtrip(golden, lmax):
    torch = cuda_or_skip()
    g = golden(f"roundtrip_l{lmax}")
    plan = _plan(lmax, g["ring_thetas"], g["ring_weights"], int(g["n_phi"]))
    assert plan.folded
    T = plan.adjoint(_t(g["a"]).reshape(1, -1), _t(g["b"]).reshape(1, -1))
    assert O.rel_l2(T[0].cpu().numpy(), g["T"]) <= TOL
    for tk, ak, bk in (("T", "fa", "fb"), ("Tn", "fna", "fnb")):
        a, b = plan.forward(_t(g[tk]).reshape(1, -1, 3))
        got = np.concatenate([a[0].cpu().numpy(), b[0].cpu().numpy()])
        assert O.rel_l2(got, np.concatenate([g[ak], g[bk]])) <= TOL
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["scattered_l16_m300", "scattered_l9_m64"])
def test_golden_scattered(golden, name):
    from paper_1908_00041_b200.plan import PointsPlan

    cuda_or_skip()
    g = golden(name)
    pp = PointsPlan(int(g["lmax"]))
    T = pp.adjoint(_t(g["points"]), _t(g["a"]).reshape(1, -1), _t(g["b"]).reshape(1, -1))
    assert O.rel_l2(T[0].cpu().numpy(), g["T"]) <= TOL


def test_reference_signature_entry_points(golden):
    import paper_1908_00041_b200 as fb

    cuda_or_skip()
    g = golden("roundtrip_l32")
    grid, rule = fb.gl_grid_for(32)
    coeffs = fb.VectorCoefficients(fb.ScalarCoefficients(32, g["a"]), fb.ScalarCoefficients(32, g["b"]))
    T = fb.adjoint_favest(coeffs, rule)
    assert O.rel_l2(T.values, g["T"]) <= TOL
    assert np.array_equal(T.points, rule.points)
    c = fb.forward_favest(T, rule, 32)
    assert O.rel_l2(np.concatenate([c.div.values, c.curl.values]), np.concatenate([g["fa"], g["fb"]])) <= 1e-10
    assert c.div.values[0] == 0 and c.curl.values[0] == 0
    # raw points -> scattered route; TensorGrid argument -> grid route
    Tp = fb.adjoint_favest(coeffs, rule.points[:100])
    assert O.rel_l2(Tp.values, g["T"][:100]) <= TOL
    Tg = fb.adjoint_favest(coeffs, grid)
    assert O.rel_l2(Tg.values, g["T"]) <= TOL
    Td = fb.adjoint_favest(coeffs, rule, path="direct-scalar")
    assert O.rel_l2(Td.values, g["T"]) <= TOL


def test_c2_batch_l256_against_oracle():
    # BASELINE configs[1]: L=256, 16 fields, 1/(l(l+1)) law, seed 2
    L, B = 256, 16
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(2)
    ab = [O.coef(rng, L, "inv") for _ in range(B)]
    A = np.stack([x[0] for x in ab])
    Bc = np.stack([x[1] for x in ab])
    plan = _plan(L, th, w, nphi, B)
    T = plan.adjoint(_t(A), _t(Bc))
    fa, fb_ = plan.forward(T)
    Tn, fa, fb_ = T.cpu().numpy(), fa.cpu().numpy(), fb_.cpu().numpy()
    from paper_1908_00041_b200.core import TangentFieldSamples
    from paper_1908_00041_b200.diagnostics import error_metrics

    pts = O.grid_points(th, nphi)
    for k in (0, 5, 15):
        Tref = O.vsht_adjoint_grid(A[k], Bc[k], L, th, nphi)
        assert O.rel_l2(Tn[k], Tref) <= TOL
        # the quadrature-weighted variant (favest/diagnostics.py:41-60) alongside
        werr, maxabs = error_metrics(TangentFieldSamples(pts, Tref), TangentFieldSamples(pts, Tn[k]),
                                     np.repeat(w, nphi))
        assert werr <= TOL and maxabs <= TOL * np.max(np.abs(Tref))
        ra, rb = O.vsht_forward_grid(Tn[k], th, w, nphi, L)
        assert O.rel_l2(np.concatenate([fa[k], fb_[k]]), np.concatenate([ra, rb])) <= TOL
    # whole batch: round trip limited by the reference's scipy GL weights
    err = O.rel_l2(np.concatenate([fa, fb_], axis=1), np.concatenate([A, Bc], axis=1))
    assert err <= 1e-10


def test_c2_field0_against_reference_fixture(golden):
    """The unmodified reference's own C2 field (L=256, tests/golden/make_golden_large.py):
    adjoint of the seeded coefficients and forward of the reference's field, every value."""
    d = golden("c2_l256_field0")
    L = int(d["lmax"])
    th, w, nphi = O.gl_grid(L)
    plan = _plan(L, th, w, nphi, 1)
    T = plan.adjoint(_t(d["a"][None]), _t(d["b"][None])).cpu().numpy()[0]
    assert O.rel_l2(T, d["T"]) <= TOL
    fa, fb_ = plan.forward(_t(d["T"][None]))
    got = np.concatenate([fa[0].cpu().numpy(), fb_[0].cpu().numpy()])
    assert O.rel_l2(got, np.concatenate([d["fa"], d["fb"]])) <= TOL


def test_c3_field0_against_reference_fixture(golden):
    """The unmodified reference at the headline size (L=1024, C3 field 0): the adjoint on 13
    rings plus per-ring sums / norms of all 1026 rings, the forward (reference run
    ring-chunked) at every degree of 24 orders plus per-order norms of all 2049 orders."""
    from test_oracle import c3_field0_inputs, order_norms

    d = golden("c3_l1024_field0")
    L = int(d["lmax"])
    a, b, rng = c3_field0_inputs(d)
    th, w, nphi = O.gl_grid(L)
    plan = _plan(L, th, w, nphi, 1)
    T = plan.adjoint(_t(a[None]), _t(b[None])).cpu().numpy()[0]
    Tr = T.reshape(L + 2, nphi, 3)
    assert O.rel_l2(Tr[d["rings"]], d["T_rings"]) <= TOL
    assert O.rel_l2(Tr.sum(axis=1), d["ring_sum"]) <= TOL
    assert np.max(np.abs(np.sqrt((np.abs(Tr) ** 2).sum(axis=(1, 2))) / d["ring_norm"] - 1)) <= TOL
    T = T + O.tangent_noise(rng, O.grid_points(th, nphi), float(d["noise_sigma"]))
    fa, fb_ = plan.forward(_t(T[None]))
    fa, fb_ = fa[0].cpu().numpy(), fb_[0].cpu().numpy()
    idx = d["flat_idx"]
    assert O.rel_l2(np.concatenate([fa[idx], fb_[idx]]), np.concatenate([d["fa_sel"], d["fb_sel"]])) <= TOL
    assert O.rel_l2(order_norms(fa, L), d["fa_order_norm"]) <= TOL
    assert O.rel_l2(order_norms(fb_, L), d["fb_order_norm"]) <= TOL


def _c3_inputs():
    L, B = 1024, 4
    rng = np.random.default_rng(3)
    ab = [O.coef(rng, L, "pow2") for _ in range(B)]
    return L, B, rng, np.stack([x[0] for x in ab]), np.stack([x[1] for x in ab])


@pytest.mark.parametrize("ptab", ["table", "on_the_fly"])
def test_c3_headline_every_order_against_oracle(ptab, monkeypatch):
    """BASELINE configs[2]: L=1024, 4 fields, (1+l)^-2 spectrum (seed 3) + tangent noise
    sigma=1e-3.  Every value of all 4 fields, adjoint and forward, against the oracle
    (run over all host cores by oracle/parallel.py), for both Legendre producers."""
    from oracle.parallel import GridPort

    torch = cuda_or_skip()
    L, B, rng, A, Bc = _c3_inputs()
    th, w, nphi = O.gl_grid(L)
    if ptab == "on_the_fly":
        monkeypatch.setenv("FV_PTAB", "0")
    plan = _plan(L, th, w, nphi, B)
    monkeypatch.delenv("FV_PTAB", raising=False)
    T = plan.adjoint(_t(A), _t(Bc)).cpu().numpy()
    pts = O.grid_points(th, nphi)
    Tin = T + np.stack([O.tangent_noise(rng, pts, 1e-3) for _ in range(B)])
    fa, fb_ = plan.forward(_t(Tin))
    fa, fb_ = fa.cpu().numpy(), fb_.cpu().numpy()
    port = GridPort(L)
    for k in range(B):
        assert O.rel_l2(T[k], port.adjoint(A[k], Bc[k])) <= TOL, k
        ra, rb = port.forward(Tin[k])
        assert O.rel_l2(np.concatenate([fa[k], fb_[k]]), np.concatenate([ra, rb])) <= TOL, k
    # size-independent property over the full batch: adjoint -> forward recovers the spectrum
    fa2, fb2 = plan.forward(_t(T))
    err = O.rel_l2(np.concatenate([fa2.cpu().numpy(), fb2.cpu().numpy()], 1), np.concatenate([A, Bc], 1))
    assert err <= 1e-10
    torch.cuda.synchronize()


def test_c4_l4096_strided_orders_and_roundtrip():
    """BASELINE configs[3] (L=4096, one field, (1+l)^-2 spectrum, seed 4) on one GPU: on-the-fly
    Legendre producer (the tables exceed the plan budget), large-prime ring DFTs (8196 = 12*683).
    Every 8th order plus the first and last 64 orders against the extended-range oracle
    (oracle/parallel.py over all host cores), adjoint in spectral space and forward, plus the
    adjoint -> forward round trip over every order."""
    from oracle.parallel import GridPort

    torch = cuda_or_skip()
    L = 4096
    Lt = L + 1
    rng = np.random.default_rng(4)
    A, Bc = O.coef(rng, L, "pow2")
    port = GridPort(L)
    th, w, nphi = port.th, port.w, port.n_phi
    plan = _plan(L, th, w, nphi, 1)
    T = plan.adjoint(_t(A[None]), _t(Bc[None]))
    orders = sorted(set(range(0, Lt + 1, 8)) | set(range(64)) | set(range(Lt + 1 - 64, Lt + 1)))
    bins = np.array(sorted({m % nphi for m in orders} | {(-m) % nphi for m in orders}))
    spec = torch.fft.fft(T[0].reshape(L + 2, nphi, 3), dim=1).div_(nphi)
    spec = spec[:, torch.from_numpy(bins).cuda()].cpu().numpy()
    ref = port.adjoint(A, Bc, orders=orders, spectrum=True)[:, bins]
    assert O.rel_l2(spec, ref) <= TOL
    del spec, ref
    fa, fb_ = plan.forward(T)
    Tn = T[0].cpu().numpy()
    del T
    out_orders = [m for m in orders if m <= L]
    ra, rb = port.forward(Tn, orders=out_orders)
    ls, ms = O.degrees_orders(L)
    sel = np.isin(np.abs(ms), out_orders)
    fa, fb_ = fa[0].cpu().numpy(), fb_[0].cpu().numpy()
    assert O.rel_l2(np.concatenate([fa[sel], fb_[sel]]), np.concatenate([ra[sel], rb[sel]])) <= TOL
    err = O.rel_l2(np.concatenate([fa, fb_]), np.concatenate([A, Bc]))
    assert err <= 1e-9  # scipy GL weights at n=4098 bound the round trip, not the kernels
    torch.cuda.synchronize()


@pytest.mark.parametrize("L", [1024, 4096])
def test_full_size_round_trip_on_the_device_rule(L):
    """Size-independent property over every order at the C3 / C4 degrees: with the
    device Gauss-Legendre rule (accurate polar weights) adjoint -> forward recovers the
    coefficients to ~1e-13; with scipy's rule the round trip is 1e-11 / 2.5e-10, the
    weights' error, not the transforms'."""
    import paper_1908_00041_b200 as fb
    from paper_1908_00041_b200.plan import GridPlan

    torch = cuda_or_skip()
    rng = np.random.default_rng(L + 7)
    a, b = O.coef(rng, L, "pow2")
    grid, _ = fb.gen_gl_tensor(2 * L + 3, on_device=True)
    plan = GridPlan.from_grid(grid, L)
    A, B = _t(a[None]), _t(b[None])
    fa, fb_ = plan.forward(plan.adjoint(A, B))
    err = float(torch.linalg.vector_norm(torch.cat([fa - A, fb_ - B], 1)) / torch.linalg.vector_norm(torch.cat([A, B], 1)))
    assert err <= 5e-12, err


def test_linearity_determinism_and_batch_consistency():
    L = 48
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(11)
    pts = O.grid_points(th, nphi)
    T1 = np.stack([O.tangent_noise(rng, pts, 1.0) for _ in range(5)])
    T2 = np.stack([O.tangent_noise(rng, pts, 1.0) for _ in range(5)])
    plan = _plan(L, th, w, nphi, 5)
    a1, b1 = plan.forward(_t(T1))
    a2, b2 = plan.forward(_t(T2))
    a3, b3 = plan.forward(_t(2.0 * T1 - 3.0 * T2))
    lhs = np.concatenate([a3.cpu().numpy(), b3.cpu().numpy()])
    rhs = np.concatenate([(2 * a1 - 3 * a2).cpu().numpy(), (2 * b1 - 3 * b2).cpu().numpy()])
    assert O.rel_l2(lhs, rhs) <= 1e-13
    a1b, b1b = plan.forward(_t(T1))
    assert bool((a1b == a1).all()) and bool((b1b == b1).all())  # bitwise reproducible
    one = _plan(L, th, w, nphi, 1)
    a4, b4 = one.forward(_t(T1[4:5]))
    assert O.rel_l2(a4.cpu().numpy(), a1[4:5].cpu().numpy()) <= 1e-15
    Ta = plan.adjoint(a1, b1)
    Tb = one.adjoint(a1[4:5].contiguous(), b1[4:5].contiguous())
    assert O.rel_l2(Tb.cpu().numpy(), Ta[4:5].cpu().numpy()) <= 1e-15


def test_adjointness_weighted_inner_product():
    # <forward(T), c> = <T, adjoint(c)>_w (the transforms are quadrature adjoints)
    L = 40
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(12)
    pts = O.grid_points(th, nphi)
    T = O.tangent_noise(rng, pts, 1.0)[None]
    a, b = O.coef(rng, L, "inv")
    plan = _plan(L, th, w, nphi)
    fa, fb_ = plan.forward(_t(T))
    S = plan.adjoint(_t(a[None]), _t(b[None])).cpu().numpy()[0]
    lhs = np.vdot(np.concatenate([a, b]), np.concatenate([fa[0].cpu().numpy(), fb_[0].cpu().numpy()]))
    wts = np.repeat(w, nphi)[:, None]
    rhs = np.vdot(S * wts, T[0])
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_odd_and_asymmetric_grids():
    import paper_1908_00041_b200 as fb

    cuda_or_skip()
    rng = np.random.default_rng(13)
    L = 10
    # odd n_theta (middle ring) and odd n_phi: gen_gl_tensor(2L+4)
    grid, _ = fb.gen_gl_tensor(2 * L + 4)
    assert grid.n_theta % 2 == 1 and grid.n_phi % 2 == 1
    # asymmetric rings -> unpaired (no equatorial folding)
    th2 = np.sort(rng.uniform(0.05, 3.0, 9))
    w2 = rng.uniform(0.01, 0.1, 9)
    for th, w, nphi, folded in ((grid.ring_thetas, grid.ring_weights, grid.n_phi, True), (th2, w2, 2 * L + 7, False)):
        plan = _plan(L, th, w, nphi)
        assert plan.folded == folded
        a, b = O.coef(rng, L, "inv")
        T = plan.adjoint(_t(a[None]), _t(b[None])).cpu().numpy()[0]
        assert O.rel_l2(T, O.vsht_adjoint_grid(a, b, L, th, nphi)) <= TOL
        Tin = T + O.tangent_noise(rng, O.grid_points(th, nphi), 0.1)
        fa, fb_ = plan.forward(_t(Tin[None]))
        ra, rb = O.vsht_forward_grid(Tin, th, w, nphi, L)
        got = np.concatenate([fa[0].cpu().numpy(), fb_[0].cpu().numpy()])
        assert O.rel_l2(got, np.concatenate([ra, rb])) <= TOL


@pytest.mark.parametrize("nphi", [24, 30, 36, 40, 42, 48, 49, 64, 75, 128, 286, 342, 2052,
                                  46, 23, 58, 86, 111, 496, 516, 984, 8196, 115, 134, 303, 1668])
def test_ring_fft_radix_plans(nphi):
    """Every packed radix (2..16 composites, primes 11..19), the small-prime
    lengths R * P with a prime 19 < P <= 64 (46 = 2 * 23, 23, 58, 86, 111 = 3 * 37,
    496 = 16 * 31, C2's 516 = 12 * 43, 984 = 24 * 41), the Rader plan (C4's
    8196 = 12 * 683), the cuFFT sub-DFT + combine path for P > 64 (134 = 2 * 67,
    303 = 3 * 101, 1668 = 12 * 139) and the cuFFT fallback (115 = 5 * 23),
    forward and adjoint against the oracle."""
    cuda_or_skip()
    rng = np.random.default_rng(nphi)
    L = 8
    th, w, _ = O.gl_grid(L)
    plan = _plan(L, th, w, nphi, B=2)
    a, b = O.coef(rng, L, "inv")
    T = plan.adjoint(_t(a[None]), _t(b[None])).cpu().numpy()[0]
    assert O.rel_l2(T, O.vsht_adjoint_grid(a, b, L, th, nphi)) <= TOL
    Tin = T + O.tangent_noise(rng, O.grid_points(th, nphi), 0.1)
    fa, fb_ = plan.forward(_t(Tin[None]))
    ra, rb = O.vsht_forward_grid(Tin, th, w, nphi, L)
    got = np.concatenate([fa[0].cpu().numpy(), fb_[0].cpu().numpy()])
    assert O.rel_l2(got, np.concatenate([ra, rb])) <= TOL


def test_c5_scattered_subset_against_oracle():
    # BASELINE configs[4]: L=128, points first then 1/(l(l+1)) coefficients, seed 5
    from paper_1908_00041_b200.plan import PointsPlan

    cuda_or_skip()
    L, M = 128, 200_000
    rng = np.random.default_rng(5)
    pts = O.random_points(rng, M)
    a, b = O.coef(rng, L, "inv")
    pp = PointsPlan(L)
    T = pp.adjoint(_t(pts), _t(a[None]), _t(b[None])).cpu().numpy()[0]
    idx = np.r_[0:12000, M - 8000:M]  # >= 20k of the 200k points
    ref = O.vsht_adjoint_points(a, b, L, pts[idx])
    assert O.rel_l2(T[idx], ref) <= TOL
    # near-pole points exercise the extended-range seeds
    polar = np.array([[0.0, 1e-9, 1.0], [1e-7, 0.0, -1.0], [0.0, 0.0, 1.0]])
    polar /= np.linalg.norm(polar, axis=1, keepdims=True)
    Tp = pp.adjoint(_t(polar), _t(a[None]), _t(b[None])).cpu().numpy()[0]
    assert O.rel_l2(Tp, O.vsht_adjoint_points(a, b, L, polar)) <= TOL


def test_api_errors_on_device():
    torch = cuda_or_skip()
    L = 8
    th, w, nphi = O.gl_grid(L)
    plan = _plan(L, th, w, nphi, 2)
    with pytest.raises(ValueError):
        plan.forward(torch.zeros((3, len(th) * nphi, 3), dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        plan.forward(torch.zeros((1, len(th) * nphi, 3), dtype=torch.complex64, device="cuda"))
    with pytest.raises(ValueError):
        plan.adjoint(torch.zeros((1, 80), dtype=torch.complex128, device="cuda"),
                     torch.zeros((1, 81), dtype=torch.complex128, device="cuda"))
    # scattered-point plans: batch above max_batch, mismatched weights, wrong dtypes
    from paper_1908_00041_b200.plan import PointsPlan

    pp = PointsPlan(L, max_batch=1)
    pts = _t(O.random_points(np.random.default_rng(0), 10))
    w = torch.ones(10, dtype=torch.float64, device="cuda")
    T2 = torch.zeros((2, 10, 3), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError, match="batch"):
        pp.forward(pts, w, T2)
    with pytest.raises(ValueError):
        pp.forward(pts, w[:9], T2[:1])
    with pytest.raises(ValueError):
        pp.forward(pts, w.float(), T2[:1])
    with pytest.raises(ValueError):
        pp.forward(pts.float(), w, T2[:1])
    # a points plan is not a grid plan and vice versa (C ABI kind checks)
    import ctypes

    lib = plan.lib
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.fv_forward_points(plan._h, pts.data_ptr(), w.data_ptr(), 10, T2.data_ptr(), T2.data_ptr(),
                                 T2.data_ptr(), 1, s) == 1
    assert b"scattered" in lib.fv_last_error()
    assert lib.fv_forward_grid(pp._h, T2.data_ptr(), T2.data_ptr(), T2.data_ptr(), 1, s) == 1


def test_host_pipeline_matches_device_path():
    """HostPipeline (overlapped pinned-host batches) returns exactly the device path's results."""
    torch = cuda_or_skip()
    from paper_1908_00041_b200.pipeline import HostPipeline

    rng = np.random.default_rng(21)
    L, B = 12, 3
    th, w, nphi = O.gl_grid(L)
    plan = _plan(L, th, w, nphi, B=B)
    A = np.stack([O.coef(rng, L, "inv")[0] for _ in range(B)])
    Bc = np.stack([O.coef(rng, L, "inv")[1] for _ in range(B)])
    T = plan.adjoint(_t(A), _t(Bc))
    fa, fb = plan.forward(T)
    T2 = plan.adjoint(fa, fb)
    pipe = HostPipeline(plan, depth=2)
    Th = torch.empty(T.shape, dtype=T.dtype, pin_memory=True)
    Th.copy_(T.cpu())
    outs = [torch.empty_like(Th, pin_memory=True) for _ in range(3)]
    for o in outs:  # three batches through two slots
        pipe.submit_roundtrip(Th, o)
    ah = torch.empty(fa.shape, dtype=fa.dtype, pin_memory=True)
    bh = torch.empty_like(ah, pin_memory=True)
    pipe.submit_forward(Th, ah, bh)
    Tadj = torch.empty_like(Th, pin_memory=True)
    Ah = torch.from_numpy(A).pin_memory()
    Bh = torch.from_numpy(Bc).pin_memory()
    pipe.submit_adjoint(Ah, Bh, Tadj)
    pipe.synchronize()
    for o in outs:
        assert torch.equal(o, T2.cpu())
    assert torch.equal(ah, fa.cpu()) and torch.equal(bh, fb.cpu())
    assert torch.equal(Tadj, T.cpu())
    with pytest.raises(ValueError):
        pipe.submit_roundtrip(T, outs[0])  # device tensor, not pinned host


@pytest.mark.parametrize("L,world,chunks", [(40, 1, 1), (40, 2, 1), (40, 3, 1), (21, 2, 1), (40, 2, 3), (21, 3, 4),
                                           (300, 4, 3), (300, 1, 1)])
def test_order_sharded_path_matches_single_plan(L, world, chunks):
    """The order-sharded building blocks (fv_ring_fft / fv_forward_orders / fv_adjoint_orders,
    dist.py) with ranks simulated in one process reproduce GridPlan.forward/adjoint, also with
    the transposes cut into order chunks; with the hand-written FFT (n_phi = 84) bitwise,
    with the cuFFT fallback (n_phi = 46) to rounding; L = 300 (5 pair chunks) with few orders
    per launch splits the forward contraction over CTAs (FwdArgs::ksplit) -- to rounding."""
    torch = cuda_or_skip()
    from paper_1908_00041_b200.dist import CudaStages, OrderShardedPlan, simulate_adjoint, simulate_forward

    rng = np.random.default_rng(L + world)
    B, maxB = 3, 4
    th, w, nphi = O.gl_grid(L)
    nth = len(th)
    plan = _plan(L, th, w, nphi, B=maxB)
    A = np.stack([O.coef(rng, L, "inv")[0] for _ in range(B)])
    Bc = np.stack([O.coef(rng, L, "inv")[1] for _ in range(B)])
    T = plan.adjoint(_t(A), _t(Bc))
    T = T + _t(np.stack([O.tangent_noise(rng, O.grid_points(th, nphi), 0.1) for _ in range(B)]))
    a_ref, b_ref = plan.forward(T)
    T_ref = plan.adjoint(a_ref, b_ref)
    plans = [OrderShardedPlan(CudaStages(plan), L, nth, nphi, maxB, r, world, plan.device, chunks=chunks)
             for r in range(world)]
    T4 = T.view(B, nth, nphi, 3)
    Tl = [T4[:, p.me.rings[0]:p.me.rings[1]].reshape(B, -1, 3).contiguous() for p in plans]
    outs = simulate_forward(plans, Tl)
    exact = nphi == 84
    for p, (a, b) in zip(plans, outs):
        sel = p.order_mask(p.me.coef)
        for x, ref in ((a, a_ref), (b, b_ref)):
            if exact:
                assert torch.equal(x[:, sel], ref[:, sel])
            else:
                assert O.rel_l2(x[:, sel].cpu().numpy(), ref[:, sel].cpu().numpy()) <= 1e-14
    Tout = simulate_adjoint(plans, outs)
    Tfull = torch.cat([t.view(B, -1, nphi, 3) for t in Tout], 1).reshape(B, -1, 3)
    if exact:
        assert torch.equal(Tfull, T_ref)
    else:
        assert O.rel_l2(Tfull.cpu().numpy(), T_ref.cpu().numpy()) <= 1e-14
    with pytest.raises(ValueError):
        plans[0].stages.lib and _lib_check_bad_orders(plan)


def _lib_check_bad_orders(plan):
    import ctypes

    from paper_1908_00041_b200 import _lib

    buf = ctypes.c_void_p(1)
    _lib.check(plan.lib.fv_forward_orders(plan._h, buf, 1, 1, 1, 0, 0, buf, buf, 1, 5, 3, 0, 0, None))


# ---------------------------------------------------------------------------
# direct-route forward at weighted points (fv_forward_points,
# favest/scalar.py:94-105 + favest/transforms.py:79-147)
# ---------------------------------------------------------------------------
def _pplan(L, B=1):
    from paper_1908_00041_b200.plan import PointsPlan

    return PointsPlan(L, max_batch=B)


def _fwd_pts(pp, pts, w, T):
    a, b = pp.forward(_t(pts), _t(w), _t(T))
    return a.cpu().numpy(), b.cpu().numpy()


@pytest.mark.parametrize("name", ["direct_gl_l12", "direct_custom_l16_m400", "direct_ico_l3"])
def test_golden_direct_forward(golden, name):
    import paper_1908_00041_b200 as fb

    cuda_or_skip()
    g = golden(name)
    L = int(g["lmax"])
    a, b = _fwd_pts(_pplan(L), g["points"], g["weights"], g["T"][None])
    ref = np.concatenate([g["fa"], g["fb"]])
    assert O.rel_l2(np.concatenate([a[0], b[0]]), ref) <= TOL
    # through the reference-signature entry point with a custom rule object
    rule = fb.QuadratureRule(points=g["points"], weights=g["weights"], exactness=0)
    c = fb.forward_favest(fb.TangentFieldSamples(g["points"], g["T"]), rule, L, path="direct-scalar")
    assert O.rel_l2(np.concatenate([c.div.values, c.curl.values]), ref) <= TOL
    assert c.div.values[0] == 0 and c.curl.values[0] == 0


def test_direct_forward_c5_points_against_oracle():
    # C5 shapes (L=128, scattered points, seeded) at a size the oracle finishes in seconds;
    # 130 degrees at m = 0, 1 exceed one 128-degree window
    cuda_or_skip()
    L, M = 128, 6000
    rng = np.random.default_rng(5)
    pts = O.random_points(rng, M)
    w = rng.uniform(0.5, 1.5, M)
    w *= 4 * np.pi / w.sum()
    T = np.stack([O.tangent_noise(rng, pts, 1.0) for _ in range(2)])
    a, b = _fwd_pts(_pplan(L, 2), pts, w, T)
    for f in range(2):
        ra, rb = O.vsht_forward_points(T[f], w, pts, L)
        assert O.rel_l2(np.concatenate([a[f], b[f]]), np.concatenate([ra, rb])) <= TOL


def test_direct_forward_multi_window_and_poles():
    # several degree windows per order (L=300), exact poles and an equator point
    cuda_or_skip()
    L, M = 300, 700
    rng = np.random.default_rng(31)
    pts = O.random_points(rng, M)
    pts[0] = [0.0, 0.0, 1.0]
    pts[1] = [0.0, 0.0, -1.0]
    pts[2] = [1.0, 0.0, 0.0]
    w = np.full(M, 4 * np.pi / M)
    T = O.tangent_noise(rng, pts, 1.0)[None]
    a, b = _fwd_pts(_pplan(L), pts, w, T)
    ra, rb = O.vsht_forward_points(T[0], w, pts, L)
    assert O.rel_l2(np.concatenate([a[0], b[0]]), np.concatenate([ra, rb])) <= TOL


def test_direct_forward_equals_grid_forward_and_is_adjoint():
    # on a GL rule the direct and FFT routes agree; <F_w T, c> = <T, S c>_w
    cuda_or_skip()
    L = 24
    th, wr, nphi = O.gl_grid(L)
    pts = O.grid_points(th, nphi)
    w = np.repeat(wr, nphi)
    rng = np.random.default_rng(17)
    T = O.tangent_noise(rng, pts, 1.0)[None]
    pp = _pplan(L)
    a, b = _fwd_pts(pp, pts, w, T)
    ga, gb = _plan(L, th, wr, nphi).forward(_t(T))
    got = np.concatenate([a[0], b[0]])
    assert O.rel_l2(got, np.concatenate([ga[0].cpu().numpy(), gb[0].cpu().numpy()])) <= 1e-12
    # adjointness at scattered points with arbitrary weights
    M = 900
    p2 = O.random_points(rng, M)
    w2 = rng.uniform(0.1, 2.0, M)
    T2 = O.tangent_noise(rng, p2, 1.0)[None]
    ca, cb = O.coef(rng, L, "inv")
    fa, fb_ = _fwd_pts(pp, p2, w2, T2)
    S = pp.adjoint(_t(p2), _t(ca[None]), _t(cb[None])).cpu().numpy()[0]
    lhs = np.vdot(np.concatenate([ca, cb]), np.concatenate([fa[0], fb_[0]]))
    rhs = np.vdot(S * w2[:, None], T2[0])
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_direct_forward_batch_determinism_and_edges():
    torch = cuda_or_skip()
    L, M = 20, 1000
    rng = np.random.default_rng(41)
    pts = O.random_points(rng, M)
    w = rng.uniform(0.5, 1.5, M)
    T = np.stack([O.tangent_noise(rng, pts, 1.0) for _ in range(5)])  # groups of 4 + 1
    pp = _pplan(L, 5)
    a, b = _fwd_pts(pp, pts, w, T)
    a2, b2 = _fwd_pts(pp, pts, w, T)
    assert np.array_equal(a, a2) and np.array_equal(b, b2)  # fixed-order reductions
    for f in (0, 4):
        sa, sb = _fwd_pts(pp, pts, w, T[f:f + 1])
        assert O.rel_l2(np.concatenate([a[f], b[f]]), np.concatenate([sa[0], sb[0]])) <= 1e-14
    # one point
    a1, b1 = _fwd_pts(pp, pts[:1], w[:1], T[:1, :1])
    ra, rb = O.vsht_forward_points(T[0, :1], w[:1], pts[:1], L)
    assert O.rel_l2(np.concatenate([a1[0], b1[0]]), np.concatenate([ra, rb])) <= TOL
    # empty rule: zero coefficients, outputs fully written
    a0 = torch.full((1, (L + 1) ** 2), 7.0, dtype=torch.complex128, device="cuda")
    b0 = a0.clone()
    pp.forward(_t(np.zeros((0, 3))), _t(np.zeros(0)), _t(np.zeros((1, 0, 3), complex)), a0, b0)
    assert float(a0.abs().max()) == 0.0 and float(b0.abs().max()) == 0.0


@pytest.mark.parametrize("nphi", [516, 8196, 46, 134, 303])
def test_ring_fft_against_numpy(nphi):
    """fv_ring_fft alone (the sharded building block) on random rings, both
    directions, against numpy's pocketfft (favest/scalar.py:149, :178); the
    large-prime lengths also through the cuFFT sub-DFT path (FV_FFT=rp) and the
    direct small-prime kernels (FV_FFT=smallp); 8196 and 516 default to the Rader
    kernels (516: several rings per CTA), 46 to the small-prime kernels."""
    import ctypes
    import os

    torch = cuda_or_skip()
    for fft in ("", "rp", "smallp"):
        os.environ["FV_FFT"] = fft
        try:
            _ring_fft_case(torch, nphi)
        finally:
            os.environ.pop("FV_FFT", None)


def _ring_fft_case(torch, nphi):
    import ctypes

    L = 8
    th, w, _ = O.gl_grid(L)
    plan = _plan(L, th, w, nphi, B=1)
    rng = np.random.default_rng(nphi + 1)
    nr = len(th)
    x = rng.standard_normal((nr, nphi, 3)) + 1j * rng.standard_normal((nr, nphi, 3))
    xd = _t(x)
    out = torch.empty((3, nr, nphi), dtype=torch.complex128, device="cuda")
    lib = plan.lib
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for inv in (0, 1):
        rc = lib.fv_ring_fft(plan._h, inv, xd.data_ptr(), 1, 3 * nphi, 3, out.data_ptr(), nr * nphi, nphi, 1, nr, s)
        assert rc == 0
        ref = np.fft.ifft(x, axis=1) * nphi if inv else np.fft.fft(x, axis=1)
        got = np.moveaxis(out.cpu().numpy(), 0, -1)
        assert O.rel_l2(got, ref) <= 1e-13


@pytest.mark.parametrize("L,B", [(100, 5), (300, 1), (400, 2), (450, 1), (700, 1)])
def test_on_the_fly_legendre_matches_table_mode(L, B):
    """FV_PTAB=0 (the on-the-fly recurrence producer; what large L uses when the
    plan tables do not fit) against the oracle and the table-mode plan, at
    forward chunk counts 2, 5, 7, 8 and 11 (32 ring pairs per chunk): every
    residue of the producer warps' tile ownership modulo 4."""
    import os

    cuda_or_skip()
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(L + B)
    A, Bc = [], []
    for _ in range(B):
        a, b = O.coef(rng, L, "inv")
        A.append(a)
        Bc.append(b)
    A, Bc = np.stack(A), np.stack(Bc)
    res = {}
    for mode in ("1", "0"):
        os.environ["FV_PTAB"] = mode
        try:
            plan = _plan(L, th, w, nphi, B=B)
        finally:
            os.environ.pop("FV_PTAB", None)
        T = plan.adjoint(_t(A), _t(Bc))
        fa, fb_ = plan.forward(T)
        res[mode] = (T.cpu().numpy(), fa.cpu().numpy(), fb_.cpu().numpy())
        del plan
    for x, y in zip(res["0"], res["1"]):
        assert O.rel_l2(x, y) <= 1e-13
    T0 = res["0"][0]
    for f in (0, B - 1):
        assert O.rel_l2(T0[f], O.vsht_adjoint_grid(A[f], Bc[f], L, th, nphi)) <= TOL
        ra, rb = O.vsht_forward_grid(T0[f], th, w, nphi, L)
        got = np.concatenate([res["0"][1][f], res["0"][2][f]])
        assert O.rel_l2(got, np.concatenate([ra, rb])) <= TOL


def test_cuda_graph_capture_replays_bitwise():
    """The C-ABI calls run on torch's current stream with no host synchronisation or
    allocation in steady state, so a round trip can be captured in a CUDA graph
    (C1 latency 56 -> 25 us, tools/c1_latency.py) and replays bitwise."""
    torch = cuda_or_skip()
    L = 32
    th, w, nphi = O.gl_grid(L)
    plan = _plan(L, th, w, nphi)
    rng = np.random.default_rng(77)
    a0, b0 = O.coef(rng, L, "inv")
    A, B = _t(a0[None]), _t(b0[None])
    T = torch.empty((1, len(th) * nphi, 3), dtype=torch.complex128, device="cuda")
    a, b = torch.empty_like(A), torch.empty_like(B)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            plan.adjoint(A, B, T)
            plan.forward(T, a, b)
    torch.cuda.synchronize()
    eager = (T.clone(), a.clone(), b.clone())
    T.zero_(); a.zero_(); b.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.adjoint(A, B, T)
        plan.forward(T, a, b)
    g.replay()
    torch.cuda.synchronize()
    for x, y in zip((T, a, b), eager):
        assert torch.equal(x, y)
    A.copy_(_t(2.0 * a0[None]))  # new inputs in the captured buffers (the transform is linear)
    B.copy_(_t(2.0 * b0[None]))
    g.replay()
    torch.cuda.synchronize()
    assert O.rel_l2(T[0].cpu().numpy(), 2.0 * eager[0][0].cpu().numpy()) <= TOL


def test_multi_group_launch_matches_single_fields():
    """Nine fields on a plan whose operand buffers hold several 4-field groups:
    two full groups go through one Legendre launch (forward and adjoint), the
    ninth field through a single-field launch; every field equals its own
    one-field transform, and the batch is bitwise reproducible."""
    L = 40
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(19)
    pts = O.grid_points(th, nphi)
    T = np.stack([O.tangent_noise(rng, pts, 1.0) for _ in range(9)])
    plan = _plan(L, th, w, nphi, 9)
    one = _plan(L, th, w, nphi, 1)
    a, b = plan.forward(_t(T))
    a2, b2 = plan.forward(_t(T))
    assert bool((a2 == a).all()) and bool((b2 == b).all())
    S = plan.adjoint(a, b)
    for f in (0, 3, 4, 7, 8):
        fa, fb_ = one.forward(_t(T[f:f + 1]))
        assert O.rel_l2(np.concatenate([a[f].cpu().numpy(), b[f].cpu().numpy()]),
                        np.concatenate([fa[0].cpu().numpy(), fb_[0].cpu().numpy()])) <= 1e-15
        Sf = one.adjoint(a[f:f + 1].contiguous(), b[f:f + 1].contiguous())
        assert O.rel_l2(S[f].cpu().numpy(), Sf[0].cpu().numpy()) <= 1e-15
    ra, rb = O.vsht_forward_grid(T[6], th, w, nphi, L)
    assert O.rel_l2(np.concatenate([a[6].cpu().numpy(), b[6].cpu().numpy()]), np.concatenate([ra, rb])) <= TOL


@pytest.mark.parametrize("L,B", [(33, 1), (100, 3), (257, 4)])
def test_adjoint_cg_runs_of_orders_bitwise_equal_to_one_order_kernel(L, B, tmp_path):
    """cg_adj_multi_kernel (runs of consecutive orders per CTA, the default) against
    cg_adj_tile_kernel (FV_CGA_MULTI=0): the same cg_adj_merge arithmetic, so the adjoint
    field must agree bitwise; the kernel choice is read once per process, hence two
    processes (tools/stage_ab.py)."""
    cuda_or_skip()
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tag, env in (("multi", {}), ("tile", {"FV_CGA_MULTI": "0"})):
        out = str(tmp_path / f"{tag}.npz")
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "stage_ab.py"), str(L), str(B), out, "1"],
                           env={**os.environ, **env}, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    for k in ("T", "fa", "fb"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


@pytest.mark.parametrize("L", [300, 450])
def test_seeded_single_field_forward_bitwise_and_split(L):
    """legendre_fwd2_kernel (plans without Legendre tables: plan-time recurrence seeds, two
    chains per producer lane, eight stages) against legendre_fwd_kernel (FV_FWD2=0): the seeds
    are the state the one-chain producer carries, so the single-field forward agrees bitwise;
    and its pair-chunk split instantiation (order-sharded launches with few orders) against
    the single plan to rounding."""
    torch = cuda_or_skip()
    from paper_1908_00041_b200.dist import CudaStages, OrderShardedPlan, simulate_forward

    th, w, nphi = O.gl_grid(L)
    nth = len(th)
    rng = np.random.default_rng(L)
    a0, b0 = O.coef(rng, L, "inv")
    plans = {}
    for tag, env in (("seeded", {"FV_PTAB": "0"}), ("plain", {"FV_PTAB": "0", "FV_FWD2": "0"})):
        os.environ.update(env)
        try:
            plans[tag] = _plan(L, th, w, nphi, B=1)
        finally:
            for k in env:
                os.environ.pop(k, None)
    T = plans["plain"].adjoint(_t(a0[None]), _t(b0[None]))
    T = T + _t(O.tangent_noise(rng, O.grid_points(th, nphi), 0.1)[None])
    fa, fb = plans["seeded"].forward(T)
    ga, gb = plans["plain"].forward(T)
    assert torch.equal(fa, ga) and torch.equal(fb, gb)
    ra, rb = O.vsht_forward_grid(T[0].cpu().numpy(), th, w, nphi, L)
    assert O.rel_l2(np.concatenate([fa[0].cpu().numpy(), fb[0].cpu().numpy()]), np.concatenate([ra, rb])) <= TOL
    world = 4
    sh = [OrderShardedPlan(CudaStages(plans["seeded"]), L, nth, nphi, 1, r, world, plans["seeded"].device, chunks=3)
          for r in range(world)]
    T4 = T.view(1, nth, nphi, 3)
    Tl = [T4[:, p.me.rings[0]:p.me.rings[1]].reshape(1, -1, 3).contiguous() for p in sh]
    for p, (a, b) in zip(sh, simulate_forward(sh, Tl)):
        sel = p.order_mask(p.me.coef)
        for x, ref in ((a, fa), (b, fb)):
            assert O.rel_l2(x[:, sel].cpu().numpy(), ref[:, sel].cpu().numpy()) <= 1e-14
