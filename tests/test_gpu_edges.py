"""Edge cases of the drop-in path on the GPU: the smallest vector degree, the
smallest admissible longitude count, empty / single-point scattered inputs,
points at the poles, and a batch that is not a multiple of the 4-field group.
Every case against the numpy oracle (relative l2 <= 1e-11)."""

import numpy as np
import pytest

import oracle as O
from gpu_util import cuda_or_skip

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _t(x):
    torch = cuda_or_skip()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("L", [1, 2, 3])
def test_smallest_degrees_round_trip(L):
    from paper_1908_00041_b200.plan import GridPlan

    cuda_or_skip()
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(300 + L)
    a, b = O.coef(rng, L, "inv")
    plan = GridPlan(L, th, w, nphi)
    T = plan.adjoint(_t(a[None]), _t(b[None])).cpu().numpy()[0]
    assert O.rel_l2(T, O.vsht_adjoint_grid(a, b, L, th, nphi)) <= TOL
    Tin = T + O.tangent_noise(rng, O.grid_points(th, nphi), 0.1)
    fa, fb = plan.forward(_t(Tin[None]))
    ra, rb = O.vsht_forward_grid(Tin, th, w, nphi, L)
    assert O.rel_l2(np.concatenate([fa[0].cpu().numpy(), fb[0].cpu().numpy()]), np.concatenate([ra, rb])) <= TOL
    assert float(abs(fa[0, 0])) == 0.0 and float(abs(fb[0, 0])) == 0.0  # l = 0 entries (favest/transforms.py:145)


@pytest.mark.parametrize("L", [5, 16])
def test_minimal_bandwidth_grid(L):
    """n_phi = 2 (L + 1) + 1, the smallest grid the fast path accepts
    (favest/transforms.py:68-72), with the GL colatitudes of the BASELINE grid."""
    from paper_1908_00041_b200.plan import GridPlan

    cuda_or_skip()
    th, w, _ = O.gl_grid(L)
    nphi = 2 * (L + 1) + 1
    w = w * (2 * L + 4) / nphi  # ring weights carry the 2 pi / n_phi factor
    rng = np.random.default_rng(400 + L)
    a, b = O.coef(rng, L, "pow2")
    plan = GridPlan(L, th, w, nphi)
    T = plan.adjoint(_t(a[None]), _t(b[None])).cpu().numpy()[0]
    assert O.rel_l2(T, O.vsht_adjoint_grid(a, b, L, th, nphi)) <= TOL
    fa, fb = plan.forward(_t(T[None]))
    ra, rb = O.vsht_forward_grid(T, th, w, nphi, L)
    assert O.rel_l2(np.concatenate([fa[0].cpu().numpy(), fb[0].cpu().numpy()]), np.concatenate([ra, rb])) <= TOL


def test_scattered_empty_single_and_polar_points():
    from paper_1908_00041_b200.plan import PointsPlan

    torch = cuda_or_skip()
    L = 20
    rng = np.random.default_rng(500)
    a, b = O.coef(rng, L, "inv")
    pp = PointsPlan(L)
    A, B = _t(a[None]), _t(b[None])
    T0 = pp.adjoint(torch.zeros((0, 3), dtype=torch.float64, device="cuda"), A, B)
    assert tuple(T0.shape) == (1, 0, 3)
    for pts in (np.array([[0.0, 0.0, 1.0]]), np.array([[0.0, 0.0, -1.0]]),
                np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0], [0.0, 0.0, -1.0], [0.6, 0.0, 0.8]])):
        got = pp.adjoint(_t(pts), A, B).cpu().numpy()[0]
        assert O.rel_l2(got, O.vsht_adjoint_points(a, b, L, pts)) <= TOL


@pytest.mark.parametrize("B", [5, 7])
def test_ragged_batch_groups(B):
    """Batches that are not a multiple of the 4-field launch group (a 4-field group
    plus a 1- or 3-field remainder) against the oracle field by field."""
    from paper_1908_00041_b200.plan import GridPlan

    cuda_or_skip()
    L = 24
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(600 + B)
    ab = [O.coef(rng, L, "inv") for _ in range(B)]
    plan = GridPlan(L, th, w, nphi, max_batch=B)
    T = plan.adjoint(_t(np.stack([x[0] for x in ab])), _t(np.stack([x[1] for x in ab]))).cpu().numpy()
    fa, fb = plan.forward(_t(T))
    for k in range(B):
        assert O.rel_l2(T[k], O.vsht_adjoint_grid(ab[k][0], ab[k][1], L, th, nphi)) <= TOL
        ra, rb = O.vsht_forward_grid(T[k], th, w, nphi, L)
        got = np.concatenate([fa[k].cpu().numpy(), fb[k].cpu().numpy()])
        assert O.rel_l2(got, np.concatenate([ra, rb])) <= TOL


@pytest.mark.parametrize("n", [1, 2, 3, 34, 515, 4098])
def test_device_gauss_legendre_rule(n):
    """fv_gauss_legendre: the n-node rule on the device against scipy's
    roots_legendre (what favest/quadrature.py:29-48 uses) and against exactness."""
    from scipy.special import roots_legendre

    from paper_1908_00041_b200.grid import gauss_legendre_device

    cuda_or_skip()
    th, w = gauss_legendre_device(n)
    nodes, gw = roots_legendre(n)
    assert np.all(np.diff(th) > 0) and th[0] > 0 and th[-1] < np.pi
    assert np.max(np.abs(np.cos(th) - nodes[::-1])) <= 4e-16 * max(1, n) ** 0.5
    assert np.max(np.abs(w / gw[::-1] - 1)[n // 4:n - n // 4 or None]) <= 1e-11  # scipy's are accurate mid-range
    assert abs(w.sum() - 2.0) <= 1e-14 * n

    def defect(x, ww):
        """max_l |sum_k w_k P_l(x_k) - 2 delta_l0| over l <= 2n - 1 (float64 recurrence)."""
        p0, p1 = np.ones(n), x.copy()
        d = max(abs(np.dot(ww, p0) - 2.0), abs(np.dot(ww, p1)))
        for l in range(2, 2 * n):
            p0, p1 = p1, ((2 * l - 1) * x * p1 - (l - 1) * p0) / l
            d = max(d, abs(np.dot(ww, p1)))
        return d

    # exactness at least as good as scipy's (measured: 6e-15 .. 2e-14 against scipy's
    # 1e-13 .. 5e-13 for n = 515 .. 4098)
    dd, ds = defect(np.cos(th), w), defect(nodes[::-1], gw[::-1])
    assert dd <= max(ds, 1e-13), (dd, ds)
    # polar weights against a 50-digit Newton (decimal): the device rule is accurate to
    # ~1e-11 where scipy's polar weights are off by 1e-9 .. 1e-7
    if n >= 100:
        for k in range(2):
            z_ref, w_ref = _gl_root_decimal(n, k)
            assert abs(np.cos(th[k]) - z_ref) <= 2e-16
            assert abs(w[k] / w_ref - 1) <= 1e-11, (k, w[k], w_ref)


def _gl_root_decimal(n, k):
    """(node, weight) of the (k+1)-th largest Gauss-Legendre node, 50-digit Newton."""
    import math
    from decimal import Decimal as D, localcontext

    with localcontext() as ctx:
        ctx.prec = 50

        def pair(z):
            p1, p0 = D(1), D(0)
            for j in range(1, n + 1):
                p2, p0 = p0, p1
                p1 = ((2 * j - 1) * z * p0 - (j - 1) * p2) / j
            return p1, p0

        z = D(math.cos(math.pi * (4 * (k + 1) - 1) / (4 * n + 2)))
        for _ in range(60):
            pn, pn1 = pair(z)
            dz = pn / (n * (z * pn - pn1) / (z * z - 1))
            z -= dz
            if abs(dz) < D(10) ** -45:
                break
        pn, pn1 = pair(z)
        dp = n * (z * pn - pn1) / (z * z - 1)
        return float(z), float(2 / ((1 - z * z) * dp * dp))


def test_device_gl_tensor_round_trip():
    """gen_gl_tensor(on_device=True) rule through the transforms: adjoint -> forward
    recovers the coefficients at least as well as with scipy's weights."""
    import paper_1908_00041_b200 as fb
    from paper_1908_00041_b200.plan import GridPlan

    cuda_or_skip()
    L = 200
    rng = np.random.default_rng(700)
    a, b = O.coef(rng, L, "inv")
    errs = []
    for dev_rule in (False, True):
        grid, rule = fb.gen_gl_tensor(2 * L + 3, on_device=dev_rule)
        assert grid.n_theta == L + 2 and len(rule) == grid.n_theta * grid.n_phi
        plan = GridPlan.from_grid(grid, L)
        T = plan.adjoint(_t(a[None]), _t(b[None]))
        fa, fb_ = plan.forward(T)
        errs.append(O.rel_l2(np.concatenate([fa[0].cpu().numpy(), fb_[0].cpu().numpy()]), np.concatenate([a, b])))
    assert errs[1] <= max(errs[0], 1e-14), errs


@pytest.mark.parametrize("L,B", [(2048, 4), (1999, 3)])
def test_large_degree_batches_fit_shared_memory(L, B):
    """Past L ~ 1900 four fields per forward launch no longer fit the kernel's shared
    memory; the plan then launches fewer fields at a time.  Batch results equal the
    single-field plan's to rounding, and the device-rule round trip holds to 5e-12."""
    import paper_1908_00041_b200 as fb
    from paper_1908_00041_b200.plan import GridPlan

    torch = cuda_or_skip()
    grid, _ = fb.gen_gl_tensor(2 * L + 3, on_device=True)
    rng = np.random.default_rng(L)
    ab = [O.coef(rng, L, "pow2") for _ in range(B)]
    A = _t(np.stack([x[0] for x in ab]))
    Bc = _t(np.stack([x[1] for x in ab]))
    plan = GridPlan.from_grid(grid, L, max_batch=B)
    T = plan.adjoint(A, Bc)
    fa, fb_ = plan.forward(T)
    err = float(torch.linalg.vector_norm(torch.cat([fa - A, fb_ - Bc], 1)) / torch.linalg.vector_norm(torch.cat([A, Bc], 1)))
    assert err <= 5e-12, err
    one = GridPlan.from_grid(grid, L, max_batch=1)
    k = B - 1
    T1 = one.adjoint(A[k:k + 1].contiguous(), Bc[k:k + 1].contiguous())
    assert float(torch.linalg.vector_norm(T1[0] - T[k]) / torch.linalg.vector_norm(T[k])) <= 1e-14
    a1, b1 = one.forward(T[k:k + 1].contiguous())
    assert float(torch.linalg.vector_norm(torch.cat([a1[0] - fa[k], b1[0] - fb_[k]])) /
                 torch.linalg.vector_norm(torch.cat([fa[k], fb_[k]]))) <= 1e-14
