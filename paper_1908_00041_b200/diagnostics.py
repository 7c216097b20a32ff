"""Transform timing records (favest/diagnostics.py:166-237) on the B200 path.

``bench`` draws the same seeded data as the reference's (same generator, same
order of draws) and times the public ``forward_favest`` / ``adjoint_favest``
calls, host arrays in and out, so a record compares one-to-one with the
reference's.  The plan for each degree (ring tables, FFT plans, Clebsch-Gordan
factors) is built by one untimed call first, as the reference builds its CG
tables outside the timer (favest/diagnostics.py:204).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .core import ScalarCoefficients, TangentFieldSamples, VectorCoefficients, flat_size
from .grid import gen_gl_tensor
from .transforms import adjoint_favest, forward_favest


def error_metrics(reference: TangentFieldSamples, reconstruction: TangentFieldSamples,
                  weights: np.ndarray) -> tuple[float, float]:
    """(relative quadrature-weighted L2 error, max pointwise Euclidean error)
    (favest/diagnostics.py:41-60); host arrays, the reference's arithmetic."""
    if reference.values.shape != reconstruction.values.shape:
        raise ValueError("sample sets have different shapes")
    w = np.asarray(weights, dtype=np.float64)
    diff = reference.values - reconstruction.values
    sq = np.sum(np.abs(diff) ** 2, axis=1)
    ref_sq = np.sum(np.abs(reference.values) ** 2, axis=1)
    num = float(np.sqrt(np.sum(w * sq)))
    den = float(np.sqrt(np.sum(w * ref_sq)))
    if den == 0.0:
        raise ValueError("reference field has zero norm")
    max_abs = float(np.max(np.sqrt(sq))) if sq.size else 0.0
    return num / den, max_abs


@dataclass
class BenchRecord:
    """Median transform timings at one degree on a tensor-grid rule."""

    lmax: int
    n_points: int
    n_coeffs: int
    forward_seconds: float
    adjoint_seconds: float
    forward_ratio: float
    adjoint_ratio: float


def bench(degrees, repetitions: int = 5, path: str = "fast-scalar", seed: int = 0,
          threads: int | None = None) -> list[BenchRecord]:
    """Median forward / adjoint times over ``repetitions`` per degree, each
    record with the ratio to the previous degree's time (nan for the first)."""
    del threads
    if repetitions < 1:
        raise ValueError("repetitions must be positive")
    rng = np.random.default_rng(seed)
    records: list[BenchRecord] = []
    for lmax in degrees:
        if lmax < 1:
            raise ValueError(f"bench degrees must be >= 1, got {lmax}")
        grid, rule = gen_gl_tensor(2 * (lmax + 1))
        values = rng.standard_normal((len(rule), 3)) + 1j * rng.standard_normal((len(rule), 3))
        samples = TangentFieldSamples(rule.points, values)
        size = flat_size(lmax)
        raw = rng.standard_normal((2, size)) + 1j * rng.standard_normal((2, size))
        raw[:, 0] = 0.0
        coeffs = VectorCoefficients(ScalarCoefficients(lmax, raw[0]), ScalarCoefficients(lmax, raw[1]))
        forward_favest(samples, rule, lmax, path=path)  # plan build, untimed
        adjoint_favest(coeffs, rule, path=path)
        fwd_times, adj_times = [], []
        for _ in range(repetitions):
            t0 = time.perf_counter()
            forward_favest(samples, rule, lmax, path=path)
            fwd_times.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            adjoint_favest(coeffs, rule, path=path)
            adj_times.append(time.perf_counter() - t0)
        fwd = float(np.median(fwd_times))
        adj = float(np.median(adj_times))
        prev = records[-1] if records else None
        records.append(BenchRecord(
            lmax=lmax, n_points=len(rule), n_coeffs=lmax * lmax + lmax,
            forward_seconds=fwd, adjoint_seconds=adj,
            forward_ratio=(fwd / prev.forward_seconds) if prev else float("nan"),
            adjoint_ratio=(adj / prev.adjoint_seconds) if prev else float("nan"),
        ))
    return records


__all__ = ["BenchRecord", "bench", "error_metrics"]
