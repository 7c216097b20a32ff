"""The drop-in entry points under concurrency and plan-cache churn (GPU)."""

import threading

import numpy as np
import pytest

import oracle as O
from gpu_util import cuda_or_skip

pytestmark = pytest.mark.gpu


def _inputs(L, n, seed):
    import paper_1908_00041_b200 as fb

    grid, rule = fb.gen_gl_tensor(2 * L + 3)
    rng = np.random.default_rng(seed)
    samples, coeffs = [], []
    for _ in range(n):
        a, b = O.coef(rng, L, "inv")
        coeffs.append(fb.VectorCoefficients(fb.ScalarCoefficients(L, a), fb.ScalarCoefficients(L, b)))
        samples.append(fb.TangentFieldSamples(rule.points, O.tangent_noise(rng, rule.points, 1.0)))
    return grid, rule, samples, coeffs


@pytest.mark.parametrize("L", [40, 300])  # 300: arrays above the stager's 4 MB direct-copy size
def test_two_threads_bitwise_equal_to_serial(L):
    import paper_1908_00041_b200 as fb

    cuda_or_skip()
    grid, rule, samples, coeffs = _inputs(L, 6, 71 + L)
    serial_f = [fb.forward_favest(s, rule, L) for s in samples]
    serial_a = [fb.adjoint_favest(c, rule) for c in coeffs]
    got_f, got_a, errs = {}, {}, []

    def work(tid):
        try:
            for rep in range(3):
                for k in range(tid, len(samples), 2):
                    got_f[(k, rep)] = fb.forward_favest(samples[k], rule, L)
                    got_a[(k, rep)] = fb.adjoint_favest(coeffs[k], rule)
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)

    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (k, _), v in got_f.items():
        assert np.array_equal(v.div.values, serial_f[k].div.values)
        assert np.array_equal(v.curl.values, serial_f[k].curl.values)
    for (k, _), v in got_a.items():
        assert np.array_equal(v.values, serial_a[k].values)
        assert v.points is rule.points or np.array_equal(v.points, rule.points)
    # results are ordinary numpy arrays the caller owns (pageable, writeable)
    assert serial_a[0].values.flags.owndata and serial_a[0].values.flags.writeable


def test_evicted_plan_stays_usable():
    import paper_1908_00041_b200 as fb
    from paper_1908_00041_b200 import transforms as tr

    torch = cuda_or_skip()
    L = 12
    grid, rule, samples, _ = _inputs(L, 1, 5)
    plan = tr.grid_plan(grid, L)
    T = torch.from_numpy(samples[0].values.reshape(1, -1, 3).copy()).cuda()
    a0, b0 = plan.forward(T)
    for k in range(tr._MAX_PLANS + 2):  # push the plan out of the cache
        g2, _ = fb.gen_gl_tensor(2 * (L + 1 + k) + 3)
        fb.forward_favest(fb.TangentFieldSamples(g2.points(), np.zeros((len(g2), 3), complex)),
                          g2.to_rule(0), L + 1 + k)
    assert plan._h is not None and plan._h.value
    a1, b1 = plan.forward(T)
    assert bool((a0 == a1).all()) and bool((b0 == b1).all())
    # a batch larger than the cached capacity replaces the cached plan, the old one lives on
    big = tr.grid_plan(grid, L, batch=3)
    assert big.max_batch >= 3 and plan._h.value
