"""Command line: the reference's ``favest bench`` (favest/cli.py:169-197,
300-314) on the GPU path.

    python -m paper_1908_00041_b200 bench --degrees 32,64,128 [--reps 5] [--seed 0] [--threads N] --out bench.csv

Exit codes as the reference's CLI (favest/cli.py:4-5): 0 on success, 2 for
usage or file errors.
"""

from __future__ import annotations

import argparse
import os
import sys


def _int_list(text: str) -> list[int]:
    return [int(tok) for tok in text.replace(",", " ").split()]


def _nonneg_int(text: str) -> int:
    v = int(text)
    if v < 0:
        raise argparse.ArgumentTypeError(f"expected a non-negative integer, got {v}")
    return v


def _resolve_threads(args) -> int:
    """favest/cli.py:43-56: --threads, else FAVEST_THREADS, else the core count."""
    value = getattr(args, "threads", None)
    if value is None:
        env = os.environ.get("FAVEST_THREADS")
        if env is not None:
            try:
                value = int(env)
            except ValueError:
                raise ValueError(f"FAVEST_THREADS is not an integer: {env!r}") from None
    if value is None:
        value = os.cpu_count() or 1
    if value < 1:
        raise ValueError(f"thread count must be >= 1, got {value}")
    return value


def cmd_bench(args) -> int:
    from .diagnostics import bench
    from .io import write_csv

    threads = _resolve_threads(args)
    records = bench(args.degrees, repetitions=args.reps, seed=args.seed, threads=threads)
    header = ("lmax", "n_points", "n_coeffs", "forward_seconds", "adjoint_seconds", "forward_ratio",
              "adjoint_ratio", "threads")
    rows = [(r.lmax, r.n_points, r.n_coeffs, r.forward_seconds, r.adjoint_seconds, r.forward_ratio,
             r.adjoint_ratio, threads) for r in records]
    write_csv(args.out, header, rows)
    print(f"wrote {len(rows)} bench rows to {args.out}")
    return 0


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="python -m paper_1908_00041_b200",
                                     description="FaVeST vector spherical harmonic transforms on B200")
    sub = parser.add_subparsers()
    threads_parent = argparse.ArgumentParser(add_help=False)
    threads_parent.add_argument("--threads", type=int, default=None)
    bn = sub.add_parser("bench", help="time forward/adjoint transforms over degrees", parents=[threads_parent])
    bn.add_argument("--degrees", type=_int_list, required=True, metavar="LIST")
    bn.add_argument("--reps", type=_nonneg_int, default=5)
    bn.add_argument("--seed", type=int, default=0)
    bn.add_argument("--out", required=True)
    bn.set_defaults(handler=cmd_bench)
    return parser


def main(argv=None) -> int:
    parser = _build_parser()
    args = parser.parse_args(argv)
    handler = getattr(args, "handler", None)
    if handler is None:
        parser.print_help(sys.stderr)
        return 2
    try:
        return handler(args)
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
