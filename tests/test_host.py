"""Host logic of the drop-in boundary: path selection, argument checks and the
error conventions of the reference (favest/transforms.py:45-76, :101-106,
favest/core.py validators).  No GPU needed: every check fires before a plan
is created."""

import numpy as np
import pytest

import paper_1908_00041_b200 as fb
from paper_1908_00041_b200 import transforms as tr
from paper_1908_00041_b200.core import ScalarCoefficients, TangentFieldSamples, VectorCoefficients


def test_gen_gl_tensor_matches_reference_bitwise(golden):
    for lmax in (8, 17, 32):
        g = golden(f"roundtrip_l{lmax}")
        grid, rule = fb.gl_grid_for(lmax)
        assert np.array_equal(grid.ring_thetas, g["ring_thetas"])
        assert np.array_equal(grid.ring_weights, g["ring_weights"])
        assert grid.n_phi == int(g["n_phi"]) == 2 * lmax + 4
        assert grid.n_theta == lmax + 2
        assert rule.grid is grid


def test_pick_path_conventions():
    grid, _ = fb.gen_gl_tensor(8)  # n_phi = 9
    with pytest.raises(ValueError, match="unknown path"):
        tr._pick_path("fastest", grid, 3)
    with pytest.raises(ValueError, match="requires a rule with tensor-grid"):
        tr._pick_path("fast-scalar", None, 3)
    with pytest.raises(ValueError, match="needs n_phi >= 11"):
        tr._pick_path("fast-scalar", grid, 4)
    assert tr._pick_path("auto", grid, 3) is True
    assert tr._pick_path("auto", grid, 4) is False
    assert tr._pick_path("direct-scalar", grid, 3) is False
    assert tr._pick_path("auto", None, 3) is False


def test_forward_argument_errors_before_any_device_work():
    grid, rule = fb.gl_grid_for(6)
    vals = np.zeros((len(rule), 3), dtype=np.complex128)
    samples = TangentFieldSamples(rule.points, vals)
    with pytest.raises(ValueError, match="lmax >= 1"):
        fb.forward_favest(samples, rule, 0)
    _, other = fb.gl_grid_for(5)
    with pytest.raises(ValueError, match="do not match"):
        fb.forward_favest(samples, other, 5)
    with pytest.raises(ValueError, match="unknown path"):
        fb.forward_favest(samples, rule, 6, path="nope")

    class Tab:
        lmax = 3

    with pytest.raises(ValueError, match="cannot serve"):
        fb.forward_favest(samples, rule, 6, tables=Tab())
    import torch

    if not torch.cuda.is_available():  # the direct route runs on the GPU only: no CPU fallback
        with pytest.raises(RuntimeError, match="needs a CUDA device"):
            fb.forward_favest(samples, rule, 6, path="direct-scalar")


def test_adjoint_argument_errors():
    c = VectorCoefficients.zeros(4)
    with pytest.raises(ValueError, match="unit sphere"):
        fb.adjoint_favest(c, np.array([[1.0, 1.0, 0.0]]))
    with pytest.raises(ValueError, match="requires a rule with tensor-grid"):
        fb.adjoint_favest(c, np.array([[1.0, 0.0, 0.0]]), path="fast-scalar")


def test_type_validators_mirror_reference():
    with pytest.raises(ValueError, match="l=0 entries"):
        VectorCoefficients(ScalarCoefficients(2, np.ones(9)), ScalarCoefficients(2, np.zeros(9)))
    with pytest.raises(ValueError, match="lmax >= 1"):
        VectorCoefficients(ScalarCoefficients(0, np.zeros(1)), ScalarCoefficients(0, np.zeros(1)))
    with pytest.raises(ValueError, match="expected 9 coefficients"):
        ScalarCoefficients(2, np.zeros(8))
    assert fb.flat_index(3, -2) == 10 and fb.flat_size(3) == 16
    with pytest.raises(ValueError):
        fb.flat_index(2, 3)


