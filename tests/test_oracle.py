"""The numpy oracle (oracle/) pinned against the reference's own outputs.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py);
known-answer values are those of the reference's tests
(pkg/tests/test_legendre.py:23-29, pkg/tests/test_coupling.py:16-20).
"""

import numpy as np
import pytest

import oracle as O
import oracle.favest_oracle as FO


def test_legendre_bitwise_against_reference(golden):
    d = golden("legendre_l40")
    p = O.legendre_table(40, d["t"])
    assert np.array_equal(p, d["p"])


def test_legendre_known_answers():
    # pkg/tests/test_legendre.py:23-29
    p = O.legendre_table(2, np.array([1.0, 0.0, -0.37]))
    assert np.allclose(p[:, O.tri_index(0, 0)], 0.28209479177387814, atol=1e-15)
    assert p[0, O.tri_index(1, 0)] == pytest.approx(0.4886025119029199, abs=1e-12)
    assert p[0, O.tri_index(1, 1)] == pytest.approx(0.0, abs=1e-15)
    assert p[1, O.tri_index(2, 0)] == pytest.approx(-0.3153915652525201, abs=1e-12)


def test_coupling_weights_known_answers():
    # pkg/tests/test_coupling.py:16-20: c_1, d_1
    assert FO._coupling_c(1) == pytest.approx(0.8164965809277260, abs=1e-15)
    assert FO._coupling_d(1) == pytest.approx(0.5773502691896258, abs=1e-15)


def test_cg_tables_bitwise_against_reference(golden):
    d = golden("cg_tables_l12")
    xi, mu = O.cg_tables(12)
    for i in range(1, 7):
        assert np.array_equal(xi[i], d[f"xi{i}"]), i
    for i in range(1, 4):
        assert np.array_equal(mu[i], d[f"mu{i}"]), i


@pytest.mark.parametrize("lmax", [8, 17, 32])
def test_grid_roundtrip_against_reference(golden, lmax):
    g = golden(f"roundtrip_l{lmax}")
    th, w, nphi = O.gl_grid(lmax)
    assert np.array_equal(th, g["ring_thetas"]) and np.array_equal(w, g["ring_weights"])
    assert nphi == int(g["n_phi"])
    T = O.vsht_adjoint_grid(g["a"], g["b"], lmax, th, nphi)
    assert O.rel_l2(T, g["T"]) <= 1e-14
    fa, fb = O.vsht_forward_grid(g["T"], th, w, nphi, lmax)
    assert O.rel_l2(np.concatenate([fa, fb]), np.concatenate([g["fa"], g["fb"]])) <= 1e-14
    fa, fb = O.vsht_forward_grid(g["Tn"], th, w, nphi, lmax)
    assert O.rel_l2(np.concatenate([fa, fb]), np.concatenate([g["fna"], g["fnb"]])) <= 1e-14


@pytest.mark.parametrize("name", ["scattered_l16_m300", "scattered_l9_m64"])
def test_scattered_adjoint_against_reference(golden, name):
    g = golden(name)
    T = O.vsht_adjoint_points(g["a"], g["b"], int(g["lmax"]), g["points"])
    assert O.rel_l2(T, g["T"]) <= 1e-14


def test_forward_is_weighted_adjoint_of_adjoint():
    # <F T, c> = <T, S c>_w for the scalar transforms (pkg/tests/test_scalar.py:72-82)
    rng = np.random.default_rng(4)
    L = 12
    th, w, nphi = O.gl_grid(L)
    N = len(th) * nphi
    f = rng.standard_normal((N, 1)) + 1j * rng.standard_normal((N, 1))
    g = rng.standard_normal((O.flat_size(L), 1)) + 1j * rng.standard_normal((O.flat_size(L), 1))
    Ff = O.sht_forward_grid(f, th, w, nphi, L)
    Sg = O.sht_adjoint_grid(g, L, th, nphi)
    lhs = np.vdot(g, Ff)
    wts = np.repeat(w, nphi)[:, None]
    rhs = np.vdot(Sg * wts, f)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_extended_range_orthonormal_at_l4096():
    # X-number recurrence stays finite and orthonormal where the reference underflows
    L = 4096
    th, w, nphi = O.gl_grid(L)
    t, s = O.ring_cos_sin(th)
    sx, se = O.seed_table(L + 1, s)
    assert se.min() < -1024  # seeds far below the double range
    gw = w * nphi / (2 * np.pi)
    for m in (1500, 4000):
        P = O.legendre_m(m, L + 1, t, sx[m], se[m])
        assert np.all(np.isfinite(P))
        G = (P * gw) @ P.T * 2 * np.pi
        assert np.max(np.abs(G - np.eye(len(G)))) < 1e-11


def test_partial_orders_match_full():
    L = 20
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(9)
    a, b = O.coef(rng, L, "inv")
    T = O.vsht_adjoint_grid(a, b, L, th, nphi)
    fa, fb = O.vsht_forward_grid(T, th, w, nphi, L)
    pa, pb = O.vsht_forward_grid(T, th, w, nphi, L, orders=[0, 5, 20])
    ls, ms = O.degrees_orders(L)
    sel = np.isin(np.abs(ms), [0, 5, 20])
    assert np.array_equal(pa[sel], fa[sel]) and np.array_equal(pb[sel], fb[sel])


@pytest.mark.parametrize("name", ["direct_gl_l12", "direct_custom_l16_m400", "direct_ico_l3"])
def test_direct_forward_against_reference(golden, name):
    # forward_favest(..., path="direct-scalar") on grid / custom / design rules
    # (favest/scalar.py:94-105, favest/transforms.py:79-147)
    g = golden(name)
    fa, fb = O.vsht_forward_points(g["T"], g["weights"], g["points"], int(g["lmax"]))
    assert O.rel_l2(np.concatenate([fa, fb]), np.concatenate([g["fa"], g["fb"]])) <= 1e-14


def test_direct_forward_matches_grid_forward():
    # on a GL rule the direct route and the FFT route are the same transform
    # (pkg/tests/test_scalar.py:96-109 pins fast == direct to 1e-11)
    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "roundtrip_l17.npz"))
    L = 17
    th, w, nphi = g["ring_thetas"], g["ring_weights"], int(g["n_phi"])
    pts = O.grid_points(th, nphi)
    fa, fb = O.vsht_forward_points(g["Tn"], np.repeat(w, nphi), pts, L)
    assert O.rel_l2(np.concatenate([fa, fb]), np.concatenate([g["fna"], g["fnb"]])) <= 1e-13


@pytest.mark.parametrize("name", ["scalar_fast_l20", "scalar_fast_l37", "scalar_fast_l1_nphi3", "scalar_fast_l0_nphi1"])
def test_scalar_grid_against_reference(golden, name):
    # forward_sht_fast / adjoint_sht_fast (favest/scalar.py:157-184)
    g = golden(name)
    L, th, w, nphi = int(g["lmax"]), g["thetas"], g["weights"], int(g["n_phi"])
    f = O.sht_adjoint_grid(g["g"][:, None], L, th, nphi)[:, 0]
    assert O.rel_l2(f, g["f"]) <= 1e-13
    fin = g["f2"] if "f2" in g else g["fr"][:, None]
    F = O.sht_forward_grid(fin, th, w, nphi, L)
    assert O.rel_l2(F, g["F"].reshape(F.shape)) <= 1e-13


def test_scalar_direct_against_reference(golden):
    # forward_sht_direct / adjoint_sht_direct (favest/scalar.py:108-128)
    g = golden("scalar_direct_l16_m400")
    L = int(g["lmax"])
    F = O.sht_forward_points(g["fr"][:, None], g["weights"], g["points"], L)[:, 0]
    assert O.rel_l2(F, g["F"]) <= 1e-13
    f = O.sht_adjoint_points(g["g"][:, None], L, g["points"])[:, 0]
    assert O.rel_l2(f, g["f"]) <= 1e-13


def test_verify_exactness_against_reference(golden):
    # favest/quadrature.py:51-76 on the icosahedron design (exact to 5), a GL
    # tensor rule (exact to 30) and a random rule, each just below and above
    g = golden("exactness")
    for name, t, d, ok in zip(g["names"], g["t"], g["defect"], g["passed"]):
        dd, okk = O.verify_exactness(g[f"{name}_points"], g[f"{name}_weights"], int(t))
        assert okk == bool(ok)
        assert abs(dd - d) <= 1e-13 + 1e-12 * d


# --------------------------------------------------------------------------
# pins at the BASELINE sizes: fixtures the unmodified reference wrote at L=256
# (the whole C2 field 0) and L=1024 (C3 field 0: 13 rings, 24 orders, and
# checksums over every ring / order), tests/golden/make_golden_large.py
# --------------------------------------------------------------------------
def c3_field0_inputs(d):
    """The C3 field-0 inputs of make_golden_large.py, regenerated from the seed:
    (a, b, noise generator positioned after the coefficients)."""
    rng = np.random.default_rng(int(d["seed"]))
    a, b = O.coef(rng, int(d["lmax"]), str(d["law"]))
    assert a.sum() == d["a_sum"] and b.sum() == d["b_sum"]  # same PCG64 stream, bitwise
    return a, b, rng


def order_norms(v, lmax):
    ls, ms = O.degrees_orders(lmax)
    out = np.zeros(2 * lmax + 1)
    np.add.at(out, ms + lmax, np.abs(v) ** 2)
    return np.sqrt(out)


def test_oracle_c2_l256_full_field_against_reference(golden):
    d = golden("c2_l256_field0")
    L = int(d["lmax"])
    rng = np.random.default_rng(int(d["seed"]))
    a, b = O.coef(rng, L, str(d["law"]))
    assert np.array_equal(a, d["a"]) and np.array_equal(b, d["b"])
    th, w, nphi = O.gl_grid(L)
    T = O.vsht_adjoint_grid(a, b, L, th, nphi)
    assert O.rel_l2(T, d["T"]) <= 1e-13
    fa, fb = O.vsht_forward_grid(d["T"], th, w, nphi, L)
    assert O.rel_l2(np.concatenate([fa, fb]), np.concatenate([d["fa"], d["fb"]])) <= 1e-13


def test_oracle_c3_l1024_against_reference(golden):
    from oracle.parallel import GridPort

    d = golden("c3_l1024_field0")
    L = int(d["lmax"])
    a, b, rng = c3_field0_inputs(d)
    port = GridPort(L)
    T = port.adjoint(a, b)
    nth, nph = L + 2, 2 * L + 4
    Tr = T.reshape(nth, nph, 3)
    assert O.rel_l2(Tr[d["rings"]], d["T_rings"]) <= 1e-13
    assert O.rel_l2(Tr.sum(axis=1), d["ring_sum"]) <= 1e-12
    assert np.max(np.abs(np.sqrt((np.abs(Tr) ** 2).sum(axis=(1, 2))) / d["ring_norm"] - 1)) <= 1e-13
    noise = O.tangent_noise(rng, O.grid_points(port.th, nph), float(d["noise_sigma"]))
    assert np.allclose(noise.sum(axis=0), d["noise_sum"], rtol=0, atol=1e-9)
    fa, fb = port.forward(T + noise)
    idx = d["flat_idx"]
    assert O.rel_l2(np.concatenate([fa[idx], fb[idx]]), np.concatenate([d["fa_sel"], d["fb_sel"]])) <= 1e-13
    for got, ref in ((order_norms(fa, L), d["fa_order_norm"]), (order_norms(fb, L), d["fb_order_norm"])):
        assert O.rel_l2(got, ref) <= 1e-13


def test_parallel_port_is_the_serial_oracle():
    from oracle.parallel import GridPort

    L = 40
    th, w, nphi = O.gl_grid(L)
    rng = np.random.default_rng(41)
    a, b = O.coef(rng, L, "pow2")
    port = GridPort(L, procs=3)
    T = port.adjoint(a, b)
    assert np.array_equal(T, O.vsht_adjoint_grid(a, b, L, th, nphi))
    fa, fb = port.forward(T)
    ra, rb = O.vsht_forward_grid(T, th, w, nphi, L)
    assert np.array_equal(fa, ra) and np.array_equal(fb, rb)
    orders = [0, 3, 17, 40]
    spec = port.adjoint(a, b, orders=orders, spectrum=True)
    ref = O.vsht_adjoint_grid(a, b, L, th, nphi, orders=orders, spectrum=True)
    assert np.array_equal(spec, ref)
    pa, pb = port.forward(T, orders=orders)
    ls, ms = O.degrees_orders(L)
    sel = np.isin(np.abs(ms), orders)
    assert np.array_equal(pa[sel], ra[sel]) and np.array_equal(pb[sel], rb[sel])
