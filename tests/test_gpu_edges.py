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
