"""Multi-GPU scan of a contiguously sharded 1-D array (one process per GPU).

Each rank holds a contiguous shard.  A rank cannot store its first output
before it knows the sum of every lower shard, so the path is Reduce-Scan-Scan
at device level (PAPER.md P73, Sec. 2.1: "the RSS approach makes a block-level
reduction first, followed by a scan of the block-level reductions and a final
scan of each block"), with GPUs as the blocks:

  1. scan_shard_reduce     one read of the shard: its sum (int64 / fp64) and the
                           sums of its 131,072-element blocks, kept on the device
  2. all_gather (NCCL)     G sums over NVLink / NVSwitch (8 bytes per rank)
  3. carry_from_totals     carry_r = totals[0] + ... + totals[r-1], fixed order
  4. scan_shard_scan       the shard scan: every block starts from carry_r + its
                           block prefix (fused into the kernel's running carry),
                           so the second read is a pure stream (row kernel)

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


PHASES = ("shard_reduce", "all_gather", "carry", "shard_scan")


def rss_scan(x_local, exclusive: bool, rank: int, world: int,
             local_total: Callable, all_gather: Callable, carry_of: Callable,
             local_scan: Callable, mark: Callable | None = None):
    """Device-level Reduce-Scan-Scan over `world` ranks (host orchestration only).

    local_total(x)             -> 1-element tensor (int64 / float64)
    all_gather(t)              -> tensor of `world` totals in rank order
    carry_of(totals, rank)     -> 1-element carry tensor
    local_scan(x, exclusive, carry) -> the rank's output shard
    mark(i)                    -> optional, called at the phase boundaries
                                  i = 0..4 (before PHASES[0] ... after PHASES[3]),
                                  e.g. to record CUDA events for per-phase timing
    """
    mark = mark or (lambda i: None)
    mark(0)
    t = local_total(x_local)
    mark(1)
    totals = all_gather(t)
    mark(2)
    carry = carry_of(totals, rank)
    mark(3)
    y = local_scan(x_local, exclusive, carry)
    mark(4)
    return y, totals, carry


def _all_gather(group):
    """All-gather of one total per rank, in rank order.  NCCL: one
    all_gather_into_tensor of G x 8 bytes over NVLink / NVSwitch, stream-ordered
    with the scan kernels.  Host backends (gloo: the multi-process tests on one
    GPU, where ranks must not exchange through device memory): the 8-byte
    totals travel through host memory."""
    backend = dist.get_backend(group)

    def gather(t):
        world = dist.get_world_size(group)
        if backend == "nccl":
            out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t, group=group)
            return out
        parts = [torch.empty(t.shape, dtype=t.dtype) for _ in range(world)]
        dist.all_gather(parts, t.cpu(), group=group)
        return torch.cat(parts).to(t.device)
    return gather


_ws_cache: dict = {}


def _shard_ws(x_local: torch.Tensor):
    """One cached workspace per (device, stream, dtype, shard length): it carries
    the block sums from pass 1 to pass 2 of a call and is reused by the next."""
    from . import shard_workspace
    key = (x_local.device.index, torch.cuda.current_stream(x_local.device).cuda_stream, x_local.dtype,
           x_local.numel())
    ws = _ws_cache.get(key)
    if ws is None:
        ws = _ws_cache[key] = shard_workspace(x_local)
    return ws


_peer_cache: dict = {}


def _peer_state(x_local: torch.Tensor, group, world: int):
    """This rank's slot array for the device-initiated exchange, in symmetric
    memory (torch.distributed._symmetric_memory: every rank's buffer mapped on
    every GPU over NVLink), with the device array of the G peer addresses."""
    from . import ScanError, peer_slots_bytes
    key = (x_local.device.index, id(group), world)
    st = _peer_cache.get(key)
    if st is None:
        try:
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(peer_slots_bytes(world) // 8, dtype=torch.int64, device=x_local.device)
            buf.zero_()
            hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
        except Exception as e:  # noqa: BLE001
            raise ScanError(f"device-initiated exchange needs symmetric memory over NVLink: {e}") from e
        torch.cuda.synchronize(x_local.device)
        dist.barrier(group)  # every slot array zeroed before anyone publishes
        st = _peer_cache[key] = {"buf": buf, "hdl": hdl, "peers": int(hdl.buffer_ptrs_dev), "epoch": 0}
    return st


def _sharded_peer(x_local, exclusive, group, out, ws, mark):
    """Reduce-Scan-Scan with the totals exchanged by the kernels themselves:
    pass 1 writes its total into every rank's slot array, pass 2 reads the
    lower ranks' totals from its own (scan.h scan_shard_reduce_publish /
    scan_shard_scan_peers) -- no NCCL call, no carry kernel."""
    from . import shard_reduce_publish, shard_scan_peers
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    st = _peer_state(x_local, group, world)
    st["epoch"] = st["epoch"] % 0xFFFFFFFF + 1  # the same sequence on every rank
    ep = st["epoch"]
    mark = mark or (lambda i: None)
    mark(0)
    shard_reduce_publish(x_local, st["peers"], world, rank, ep, ws=ws)
    mark(1)
    mark(2)  # the exchange is inside the two kernels
    mark(3)
    y = shard_scan_peers(x_local, exclusive, st["buf"], world, rank, ep, ws=ws, out=out)
    mark(4)
    return y


def _sharded(x_local: torch.Tensor, exclusive: bool, group=None, out=None, ws=None, mark=None,
             exchange: str = "nccl"):
    from . import carry_from_totals, shard_reduce, shard_scan
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ws = ws if ws is not None else _shard_ws(x_local)
    if exchange == "peer":
        return _sharded_peer(x_local, exclusive, group, out, ws, mark)

    def local_scan(x, exc, carry):
        return shard_scan(x, exc, carry_in=carry, ws=ws, out=out)

    y, _, _ = rss_scan(x_local, exclusive, rank, world,
                       local_total=lambda x: shard_reduce(x, ws=ws),
                       all_gather=_all_gather(group),
                       carry_of=lambda totals, r: carry_from_totals(totals, r, x_local.dtype),
                       local_scan=local_scan, mark=mark)
    return y


def sharded_inclusive(x_local: torch.Tensor, group=None, out=None, ws=None, mark=None,
                      exchange: str = "nccl") -> torch.Tensor:
    """Inclusive scan of the array whose rank-r contiguous shard is x_local
    (`ws`: a reusable paper_2505_15112_b200.shard_workspace for this shard;
    `mark`: see rss_scan; exchange="peer": the device-initiated totals
    exchange over symmetric memory instead of the NCCL all-gather)."""
    return _sharded(x_local, False, group, out, ws, mark, exchange)


def sharded_exclusive(x_local: torch.Tensor, group=None, out=None, ws=None, mark=None,
                      exchange: str = "nccl") -> torch.Tensor:
    """Exclusive scan of the array whose rank-r contiguous shard is x_local."""
    return _sharded(x_local, True, group, out, ws, mark, exchange)
