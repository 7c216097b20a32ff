"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
(read-only; nothing is copied) and writes small .npz fixtures next to this
script.  The fixtures pin both the numpy oracle (tests/test_oracle.py) and
the CUDA path (tests/test_gpu_parity.py) to the reference's own outputs.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import favest
    from favest.core import ScalarCoefficients, TangentFieldSamples, VectorCoefficients, degrees_orders
    from favest.coupling import build_cg_tables
    from favest.legendre import legendre_table
    from favest.quadrature import gen_gl_tensor
    from favest.transforms import adjoint_favest, forward_favest

    def coef(rng, lmax, law):
        K = (lmax + 1) ** 2
        ls, _ = degrees_orders(lmax)
        lf = ls.astype(np.float64)
        if law == "inv":
            scale = np.where(ls >= 1, 1.0 / np.maximum(lf * (lf + 1.0), 1.0), 0.0)
        else:
            scale = (1.0 + lf) ** -2
        out = []
        for _ in range(2):
            v = (rng.standard_normal(K) + 1j * rng.standard_normal(K)) * scale
            v[0] = 0.0
            out.append(v)
        return out

    def vc(a, b, lmax):
        return VectorCoefficients(ScalarCoefficients(lmax, a), ScalarCoefficients(lmax, b))

    # 1. Legendre values (bitwise pin of the recurrence) on a GL ring set and frozen args
    grid, _ = gen_gl_tensor(2 * 38 + 3)
    t = np.concatenate([np.cos(grid.ring_thetas), [1.0, 0.0, -0.37]])
    np.savez_compressed(os.path.join(HERE, "legendre_l40.npz"), t=t, p=legendre_table(40, t))

    # 2. CG tables (bitwise pin of the closed forms)
    tab = build_cg_tables(12)
    np.savez_compressed(
        os.path.join(HERE, "cg_tables_l12.npz"),
        **{f"xi{i}": tab.xi[i] for i in range(1, 7)},
        **{f"mu{i}": tab.mu[i] for i in range(1, 4)},
    )

    # 3. grid round trips: C1 (L=32, seed 1, 1/(l(l+1)) law) plus odd/small L
    for lmax, seed in ((32, 1), (8, 101), (17, 117)):
        grid, rule = gen_gl_tensor(2 * lmax + 3)
        rng = np.random.default_rng(seed)
        a, b = coef(rng, lmax, "inv")
        tables = build_cg_tables(lmax)
        T = adjoint_favest(vc(a, b, lmax), rule, tables=tables)
        F = forward_favest(T, rule, lmax, tables=tables)
        # a noisy (non-bandlimited) tangent field through the forward
        pts = rule.points
        raw = 1e-3 * (rng.standard_normal(pts.shape) + 1j * rng.standard_normal(pts.shape))
        raw -= np.sum(raw * pts, axis=1)[:, None] * pts
        Tn = TangentFieldSamples(pts, T.values + raw)
        Fn = forward_favest(Tn, rule, lmax, tables=tables)
        np.savez_compressed(
            os.path.join(HERE, f"roundtrip_l{lmax}.npz"),
            lmax=lmax, ring_thetas=grid.ring_thetas, ring_weights=grid.ring_weights,
            n_phi=grid.n_phi, a=a, b=b, T=T.values, fa=F.div.values, fb=F.curl.values,
            Tn=Tn.values, fna=Fn.div.values, fnb=Fn.curl.values,
        )

    # 4. scattered-point adjoint (direct route), C5 recipe at small size
    for lmax, M, seed in ((16, 300, 5), (9, 64, 55)):
        rng = np.random.default_rng(seed)
        v = rng.standard_normal((M, 3))
        pts = v / np.linalg.norm(v, axis=1, keepdims=True)
        a, b = coef(rng, lmax, "inv")
        out = adjoint_favest(vc(a, b, lmax), pts)
        np.savez_compressed(
            os.path.join(HERE, f"scattered_l{lmax}_m{M}.npz"),
            lmax=lmax, points=pts, a=a, b=b, T=out.values,
        )
    # 5. direct-route forward on non-grid rules (favest/scalar.py:94-105):
    #    (a) a GL tensor rule forced onto path="direct-scalar",
    #    (b) a custom rule: random points, random positive weights summing to 4 pi,
    #    (c) the bundled 12-point icosahedron design (equal weights 4 pi / 12)
    from favest.core import QuadratureRule
    from favest.quadrature import bundled_design

    def tangent(rng, pts, scale=1.0):
        raw = scale * (rng.standard_normal(pts.shape) + 1j * rng.standard_normal(pts.shape))
        return raw - np.sum(raw * pts, axis=1)[:, None] * pts

    cases = []
    grid, rule = gen_gl_tensor(2 * 12 + 3)
    rng = np.random.default_rng(121)
    a, b = coef(rng, 12, "inv")
    T = adjoint_favest(vc(a, b, 12), rule)
    cases.append(("direct_gl_l12", 12, rule, T.values + tangent(rng, rule.points, 1e-3)))
    rng = np.random.default_rng(161)
    M = 400
    v = rng.standard_normal((M, 3))
    pts = v / np.linalg.norm(v, axis=1, keepdims=True)
    w = rng.uniform(0.5, 1.5, M)
    w *= 4.0 * np.pi / w.sum()
    rule = QuadratureRule(points=pts, weights=w, exactness=0)
    cases.append(("direct_custom_l16_m400", 16, rule, tangent(rng, pts)))
    rule = bundled_design("icosahedron12")
    rng = np.random.default_rng(12)
    cases.append(("direct_ico_l3", 3, rule, tangent(rng, rule.points)))
    for name, lmax, rule, vals in cases:
        F = forward_favest(TangentFieldSamples(rule.points, vals), rule, lmax, path="direct-scalar")
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            lmax=lmax, points=rule.points, weights=rule.weights, T=vals,
            fa=F.div.values, fb=F.curl.values,
        )
    # 6. scalar transforms (favest/scalar.py:108-184) and rule certification
    #    (favest/quadrature.py:51-76).  ScalarCoefficients holds one column
    #    (favest/core.py:104-112), so the public calls take one field each;
    #    f2's three columns are transformed one by one (the plan-level batch
    #    is checked against them).
    from favest.scalar import TensorGrid, adjoint_sht_direct, adjoint_sht_fast, forward_sht_direct, forward_sht_fast
    from favest.quadrature import verify_exactness

    def scoef(rng, lmax, c=None):
        K = (lmax + 1) ** 2
        shape = (K,) if c is None else (K, c)
        ls, _ = degrees_orders(lmax)
        scale = (1.0 + ls.astype(np.float64)) ** -1.5
        if c is not None:
            scale = scale[:, None]
        return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * scale

    rng = np.random.default_rng(2024)
    for lmax, t in ((20, 41), (37, 80)):
        grid, rule = gen_gl_tensor(t)
        g = scoef(rng, lmax)
        f = adjoint_sht_fast(ScalarCoefficients(lmax, g), grid)
        f2 = np.stack([f + 1e-3 * (rng.standard_normal(f.shape) + 1j * rng.standard_normal(f.shape)),
                       rng.standard_normal(f.shape) + 0j, f.conj()], axis=1)
        F = np.stack([forward_sht_fast(f2[:, c], grid, lmax).values for c in range(3)], axis=1)
        np.savez_compressed(
            os.path.join(HERE, f"scalar_fast_l{lmax}.npz"),
            lmax=lmax, thetas=grid.ring_thetas, weights=grid.ring_weights, n_phi=grid.n_phi,
            g=g, f=f, f2=f2, F=F,
        )
    # tiny rings: n_phi = 3 with lmax = 1, n_phi = 1 with lmax = 0
    for lmax, n_phi in ((1, 3), (0, 1)):
        grid = TensorGrid(ring_thetas=np.array([0.4, 1.3, 2.2]), ring_weights=np.array([0.7, 1.9, 0.8]) / n_phi,
                          n_phi=n_phi)
        g = scoef(rng, lmax)
        f = adjoint_sht_fast(ScalarCoefficients(lmax, g), grid)
        fr = rng.standard_normal(f.shape) + 1j * rng.standard_normal(f.shape)
        F = forward_sht_fast(fr, grid, lmax).values
        np.savez_compressed(
            os.path.join(HERE, f"scalar_fast_l{lmax}_nphi{n_phi}.npz"),
            lmax=lmax, thetas=grid.ring_thetas, weights=grid.ring_weights, n_phi=n_phi, g=g, f=f, fr=fr, F=F,
        )
    rng = np.random.default_rng(4001)
    M, lmax = 400, 16
    v = rng.standard_normal((M, 3))
    pts = v / np.linalg.norm(v, axis=1, keepdims=True)
    w = rng.uniform(0.5, 1.5, M)
    w *= 4.0 * np.pi / w.sum()
    rule = QuadratureRule(points=pts, weights=w, exactness=0)
    fr = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    F = forward_sht_direct(fr, rule, lmax).values
    g = scoef(rng, lmax)
    f = adjoint_sht_direct(ScalarCoefficients(lmax, g), pts)
    np.savez_compressed(os.path.join(HERE, "scalar_direct_l16_m400.npz"),
                        lmax=lmax, points=pts, weights=w, fr=fr, F=F, g=g, f=f)
    ico = bundled_design("icosahedron12")
    _, glr = gen_gl_tensor(30)
    rows = []
    for name, r, t in (("ico", ico, 5), ("ico", ico, 6), ("ico", ico, 0), ("gl30", glr, 30), ("gl30", glr, 31),
                       ("custom", rule, 4)):
        d, ok = verify_exactness(r, t)
        rows.append((name, t, d, ok))
    np.savez_compressed(os.path.join(HERE, "exactness.npz"),
                        names=np.array([r[0] for r in rows]), t=np.array([r[1] for r in rows]),
                        defect=np.array([r[2] for r in rows]), passed=np.array([r[3] for r in rows]),
                        ico_points=ico.points, ico_weights=ico.weights, gl30_points=glr.points,
                        gl30_weights=glr.weights, custom_points=pts, custom_weights=w)
    # 7. file formats (favest/io.py, favest/quadrature.py:79-139): files the
    #    reference writers produce, and malformed inputs with the exception
    #    type and message the reference readers raise ("{path}" for the name)
    import json
    import tempfile

    from favest import io as rio
    from favest.quadrature import load_design

    iodir = os.path.join(HERE, "io")
    os.makedirs(iodir, exist_ok=True)
    rng = np.random.default_rng(7007)
    L = 12
    a, b = coef(rng, L, "inv")
    b[3] = 1e16 + 0.5j
    b[4] = complex(-0.0, 5e-324)
    b[5] = complex(1.7976931348623157e308, -2.2250738585072014e-308)
    rio.write_coefficients(os.path.join(iodir, "coef_l12.json"), vc(a, b, L))
    grid, rule = gen_gl_tensor(13)
    rio.write_rule_file(os.path.join(iodir, "gl13.rule"), rule)
    vals = tangent(rng, rule.points)
    rio.write_samples(os.path.join(iodir, "samples_gl13.csv"), TangentFieldSamples(rule.points, vals))
    rio.write_csv(os.path.join(iodir, "table.csv"), ("l", "err", "name"),
                  [(1, 0.1, "x"), (2, 1e-300, "y")])
    rio.write_csv(os.path.join(iodir, "table_f.csv"), ("x", "y"), [(0.1, 2.5), (1e-300, -3.0)])
    np.savez_compressed(os.path.join(iodir, "values.npz"), a=a, b=b, points=rule.points,
                        weights=rule.weights, vals=vals)

    good_pair = "[[0, 0], [1, 2], [3, 4], [5, 6]]"
    cases = [
        ("coef", "not json", "{"),
        ("coef", "extra data", '{"L_max": 1, "a": [], "b": []} x'),
        ("coef", "missing b", '{"L_max": 1, "a": ' + good_pair + "}"),
        ("coef", "top list", "[1, 2]"),
        ("coef", "wrong len", '{"L_max": 1, "a": [[0, 0]], "b": ' + good_pair + "}"),
        ("coef", "lmax float", '{"L_max": 1.9, "a": ' + good_pair + ', "b": ' + good_pair + "}"),
        ("coef", "lmax string", '{"L_max": "1", "a": ' + good_pair + ', "b": ' + good_pair + "}"),
        ("coef", "lmax bad string", '{"L_max": "x", "a": [], "b": []}'),
        ("coef", "lmax negative", '{"L_max": -2, "a": [], "b": []}'),
        ("coef", "string values", '{"L_max": 1, "a": [[0, 0], ["1_0.5", " -2e3 "], [0, 0], [0, 0]], '
                              '"b": [[0, 0], ["inf", "-NaN"], [" +.5", "5."], ["1E-2", "-Infinity"]]}'),
        ("coef", "bad string value", '{"L_max": 0, "a": [["1..5", 0]], "b": [[0, 0]]}'),
        ("coef", "null value", '{"L_max": 0, "a": [[null, 0]], "b": [[0, 0]]}'),
        ("coef", "triple", '{"L_max": 0, "a": [[1, 2, 3]], "b": [[0, 0]]}'),
        ("coef", "single", '{"L_max": 0, "a": [[1]], "b": [[0, 0]]}'),
        ("coef", "number pair", '{"L_max": 0, "a": [5], "b": [[0, 0]]}'),
        ("coef", "string pairs", '{"L_max": 1, "a": [[0, 0], "12", "00", [1, 1]], "b": [[0, 0], "12", "00", "7"]}'),
        ("coef", "dict pair", '{"L_max": 1, "a": [[0, 0], {"1": 0, "2": 0}, [0, 0], [1, 1]], "b": ' + good_pair + "}"),
        ("coef", "string pair ok", '{"L_max": 1, "a": [[0, 0], "12", {"3": 0, "4": 0}, [1, 1]], "b": ' + good_pair + "}"),
        ("coef", "json literals", '{"L_max": 1, "a": [[0, 0], [NaN, Infinity], [0, 0], [0, 0]], '
                              '"b": [[0, 0], [-Infinity, true], [false, 0], [0, 0]]}'),
        ("coef", "duplicate key", '{"L_max": 3, "L_max": 1, "a": [[1, 2]], "b": ' + good_pair
         + ', "a": ' + good_pair.replace("1", "7") + "}"),
        ("coef", "python nan", '{"L_max": 0, "a": [[nan, 0]], "b": [[0, 0]]}'),
        ("coef", "big ints", '{"L_max": 1, "a": [[0, 0], [12345678901234567890123, -0], [0, 0], [0, 0]], '
                         '"b": [[0, 0], [1e400, 1e-400], [-0.0, 4.9e-324], [0, 0]]}'),
        ("rule", "ragged", "0 0 1 1\n1 0 0\n"),
        ("rule", "two cols", "0 0\n1 0\n"),
        ("rule", "bad float", "0 0 1\n1 0 x\n"),
        ("rule", "empty", "# nothing\n\n"),
        ("rule", "off sphere", "0 0 1.1\n1 0 0\n"),
        ("rule", "commas and crlf", "# c\r\n0, 0, 1 # x\r\n1,0,0\r\n0 1 0\r0 0 -1\n1e0 0 0\n0 -1 0\n"),
        ("rule", "underscores", "0 0 1_0\n1 0 0\n"),
        ("samples", "seven cols", "theta,phi,a,b,c,d,e,f\n1,2,3,4,5,6,7\n"),
        ("samples", "bad float", "1,2,3,4,5,6,7,zz\n"),
        ("samples", "empty", "theta,phi,t1_re,t1_im,t2_re,t2_im,t3_re,t3_im\n"),
        ("samples", "comments quoted", '# hi\n"1.0",2,3,4,5,6,7,8\n\n 0.5 ,1,0,0,0,0,0,0\r\n'),
        ("samples", "header later", "1,2,3,4,5,6,7,8\ntheta,phi,a,b,c,d,e,f\n"),
    ]
    results = []
    tmpd = tempfile.mkdtemp()
    for kind, name, text in cases:
        path = os.path.join(tmpd, "case.txt")
        with open(path, "w", newline="") as fh:
            fh.write(text)
        try:
            if kind == "coef":
                c = rio.read_coefficients(path)
                out = {"ok": True, "lmax": c.lmax,
                       "a": [[float(v.real), float(v.imag)] for v in c.div.values],
                       "b": [[float(v.real), float(v.imag)] for v in c.curl.values]}
            elif kind == "rule":
                r = rio.read_rule_file(path, 1)
                out = {"ok": True, "points": r.points.tolist(), "weights": r.weights.tolist(), "kind": r.kind}
            else:
                s = rio.read_samples(path)
                out = {"ok": True, "points": s.points.tolist(),
                       "values": [[[float(v.real), float(v.imag)] for v in row] for row in s.values]}
        except Exception as exc:  # noqa: BLE001 - the fixture records the reference's exception
            out = {"ok": False, "type": type(exc).__name__, "msg": str(exc).replace(path, "{path}")}
        results.append({"kind": kind, "name": name, "text": text, "out": out})
    design = os.path.join(tmpd, "design.txt")
    with open(design, "w") as fh:
        fh.write("# octahedron\n1 0 0\n-1 0 0\n0 1 0\n0 -1 0\n0 0 1\n0 0 -1.0000000001\n")
    d = load_design(design, 3)
    results.append({"kind": "design", "name": "octahedron", "text": open(design).read(),
                    "out": {"ok": True, "points": d.points.tolist(), "weights": d.weights.tolist(), "kind": d.kind}})
    with open(os.path.join(iodir, "cases.json"), "w") as fh:
        json.dump(results, fh, indent=1, allow_nan=True)
    print("reference favest", getattr(favest, "__version__", "?"), "numpy", np.__version__)


if __name__ == "__main__":
    main()
