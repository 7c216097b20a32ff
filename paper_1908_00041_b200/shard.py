"""Work partitioning across GPUs (one process per GPU, torch.distributed).

Two ways the VSHT shards:

* by field batch — fields are independent; each rank transforms its own
  slice with no data-path collective (weak scaling, used by ``bench.py``);
* by spherical-harmonic order m — the per-order Legendre work is
  proportional to (L+2-m); ``order_blocks`` gives every rank two mirror-image
  blocks [m0, m1) and [Lt+1-m1, Lt+1-m0) so all ranks get equal area, the
  layout the NCCL all-to-all transpose (ring-major FFT output -> m-major) of the
  m-sharded path uses.

Everything here is host logic; it is exercised with world_size-2 gloo tests.
"""

from __future__ import annotations


def shard_batch(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of B fields for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if B < 0:
        raise ValueError("negative batch")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def order_work(Lt: int, m: int) -> int:
    """Legendre work of order m at scalar degree Lt: number of degrees l in [m, Lt]."""
    return max(0, Lt + 1 - m)


def order_blocks(Lt: int, world: int) -> list[list[int]]:
    """Orders 0..Lt split into ``world`` sets of (near) equal total work.

    Pairs m with Lt-m ("zig-zag"): each pair carries Lt+2 units of work (a
    middle singleton less); pairs are dealt greedily to the least-loaded rank,
    which balances to within one pair.  Returns the sorted order list of every rank.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    n = Lt + 1
    pairs = [(m, Lt - m) for m in range((n + 1) // 2)]
    per = [[] for _ in range(world)]
    load = [0] * world
    for a, b in pairs:
        r = min(range(world), key=lambda k: (load[k], k))
        per[r].append(a)
        load[r] += order_work(Lt, a)
        if b != a:
            per[r].append(b)
            load[r] += order_work(Lt, b)
    return [sorted(x) for x in per]


def rank_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    import os

    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))
