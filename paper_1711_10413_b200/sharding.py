"""Config 5: the team grid / element range sharded across GPUs.

Teams are independent (per-team state lives in each CTA's shared memory and
cross-team access is forbidden, Simulator.cpp:336-351), so GPU g owns the
contiguous element range [g*N/G, (g+1)*N/G) and its own teams, with the cyclic
schedule inside each GPU.  There is no data-path collective: after the region
the per-GPU checksums (sum of the elements' bit patterns mod 2^64) are
gathered once with an all-reduce, exact for any world size because the two
32-bit halves are reduced separately.
"""
from __future__ import annotations

from typing import Tuple

MASK64 = (1 << 64) - 1


def shard_range(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """[lo, hi) of the elements owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * n_total // world, (rank + 1) * n_total // world


def split64(c: int):
    c &= MASK64
    return c & 0xFFFFFFFF, c >> 32


def join64(lo_sum: int, hi_sum: int) -> int:
    return (lo_sum + (hi_sum << 32)) & MASK64


def allreduce_checksum(local: int, device=None) -> int:
    """Sum of every rank's 64-bit checksum mod 2^64 over torch.distributed."""
    import torch
    import torch.distributed as dist
    lo, hi = split64(local)
    t = torch.tensor([lo, hi], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return join64(int(t[0].item()), int(t[1].item()))
