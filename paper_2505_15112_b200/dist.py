"""Multi-GPU scan of a contiguously sharded 1-D array (one process per GPU).

Each rank holds a contiguous shard.  A rank cannot store its first output
before it knows the sum of every lower shard, so the path is Reduce-Scan-Scan
at device level (PAPER.md P73, Sec. 2.1: "the RSS approach makes a block-level
reduction first, followed by a scan of the block-level reductions and a final
scan of each block"), with GPUs as the blocks:

  1. scan_total            the shard's sum (int64 / fp64), one read of the shard
  2. all_gather (NCCL)     G sums over NVLink / NVSwitch (8 bytes per rank)
  3. carry_from_totals     carry_r = totals[0] + ... + totals[r-1], fixed order
  4. scan_inclusive/excl.  the shard scan, seeded with carry_r (fused into the
                           kernel's block carries, so no extra pass)

The host logic (shard bounds, the order of the exchange, the carry
composition) lives in `rss_scan`, which takes the per-rank operations as
arguments: the product binds them to the CUDA library (`sharded_inclusive`
/ `sharded_exclusive`); the CPU tests bind them to the oracle over gloo.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard r of n elements: [r*ceil(n/G), min(n, (r+1)*ceil(n/G)))."""
    per = -(-n // world) if world > 0 else 0
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


def rss_scan(x_local, exclusive: bool, rank: int, world: int,
             local_total: Callable, all_gather: Callable, carry_of: Callable,
             local_scan: Callable):
    """Device-level Reduce-Scan-Scan over `world` ranks (host orchestration only).

    local_total(x)             -> 1-element tensor (int64 / float64)
    all_gather(t)              -> tensor of `world` totals in rank order
    carry_of(totals, rank)     -> 1-element carry tensor
    local_scan(x, exclusive, carry) -> the rank's output shard
    """
    t = local_total(x_local)
    totals = all_gather(t)
    carry = carry_of(totals, rank)
    return local_scan(x_local, exclusive, carry), totals, carry


def _nccl_all_gather(group):
    def gather(t):
        world = dist.get_world_size(group)
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    return gather


def _sharded(x_local: torch.Tensor, exclusive: bool, group=None, out=None):
    from . import carry_from_totals, exclusive as scan_exc, inclusive as scan_inc, total
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)

    def local_scan(x, exc, carry):
        return (scan_exc if exc else scan_inc)(x, out=out, carry_in=carry)

    y, _, _ = rss_scan(x_local, exclusive, rank, world,
                       local_total=total,
                       all_gather=_nccl_all_gather(group),
                       carry_of=lambda totals, r: carry_from_totals(totals, r, x_local.dtype),
                       local_scan=local_scan)
    return y


def sharded_inclusive(x_local: torch.Tensor, group=None, out=None) -> torch.Tensor:
    """Inclusive scan of the array whose rank-r contiguous shard is x_local."""
    return _sharded(x_local, False, group, out)


def sharded_exclusive(x_local: torch.Tensor, group=None, out=None) -> torch.Tensor:
    """Exclusive scan of the array whose rank-r contiguous shard is x_local."""
    return _sharded(x_local, True, group, out)
