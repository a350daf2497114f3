"""The PRODUCT multi-GPU path (paper_2505_15112_b200.dist.sharded_inclusive /
sharded_exclusive -> scan_shard_reduce -> all-gather -> scan_carry_from_totals
-> scan_shard_scan) run by 2 and 3 real processes, each one rank of a
process group, against the oracle over the whole array.

Only one GPU is available, so every rank drives cuda:0 and the group is gloo:
the 8-byte totals travel through host memory (dist._all_gather's host branch),
so no rank's kernel ever waits on another rank's kernel (B200_PROFILING.md:
ranks that wait on one another must not share one GPU).  Everything else --
shard bounds, the per-rank workspaces, the carry composition, both CUDA passes
-- is the code bench.py runs over NCCL.  Integers bit-exact (C3-type int8
flags), floats within the north_star tolerance (C5-type N(0,1) fp32)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, kind, seed, exclusive, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import inputs
        import paper_2505_15112_b200 as S
        from paper_2505_15112_b200 import dist as D
        S.load()
        lo, hi = D.shard_bounds(n, world, rank)
        x = inputs.fill_host(kind, seed, lo, hi - lo)
        xd = torch.from_numpy(x)
        if kind == inputs.F16_U01:
            xd = xd.view(torch.float16)
        xd = xd.cuda()
        fn = D.sharded_exclusive if exclusive else D.sharded_inclusive
        outs = []
        for _ in range(2):  # twice: the cached shard workspace is reused
            outs.append(fn(xd).cpu().numpy())
        torch.cuda.synchronize()
        q.put((rank, lo, hi, outs, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, 0, 0, None, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run(world, n, kind, seed, exclusive):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, kind, seed, exclusive, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errs = [r[4] for r in res if r[4]]
    assert not errs, errs
    return sorted(res)


@pytest.mark.parametrize("world", [2, 3])
def test_product_sharded_int8_flags_exclusive(oracle, inputs_mod, world):
    n = (1 << 24) + 12345  # several 131,072-element blocks per shard, ragged shard tails
    res = _run(world, n, inputs_mod.I8_FLAG, 2, True)
    x = inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n)
    ref = oracle.exclusive(x, "i8")
    for rank, lo, hi, outs, _ in res:
        for y in outs:
            assert np.array_equal(y, ref[lo:hi]), (world, rank)


@pytest.mark.parametrize("world", [2, 3])
def test_product_sharded_fp32_inclusive(oracle, inputs_mod, world):
    n = (1 << 22) + 777
    res = _run(world, n, inputs_mod.F32_NORMAL, 4, False)
    x = inputs_mod.fill_host(inputs_mod.F32_NORMAL, 4, 0, n)
    y64, a64, _ = oracle.inclusive(x, "f32")
    for rank, lo, hi, outs, _ in res:
        for y in outs:
            bad, worst, at = oracle.check_f32(y, y64[lo:hi], a64[lo:hi])
            assert bad == 0, (world, rank, worst, at)


def test_product_sharded_fp16_inclusive(oracle, inputs_mod):
    n = (1 << 23) + 3
    res = _run(2, n, inputs_mod.F16_U01, 1, False)
    x = inputs_mod.fill_host(inputs_mod.F16_U01, 1, 0, n)
    y64, a64, _ = oracle.inclusive(x, "f16")
    for rank, lo, hi, outs, _ in res:
        for y in outs:
            bad, worst, at = oracle.check_f32(y, y64[lo:hi], a64[lo:hi])
            assert bad == 0, (rank, worst, at)


# ------------------------------------------------------------------ device-initiated exchange

def _emulated_peer_exchange(cuda, x_shards, exclusive, G, epochs):
    """G ranks emulated in ONE process on cuda:0 (B200_PROFILING.md: with fewer
    GPUs than ranks, no rank's kernel may wait on another's concurrently): every
    rank's pass 1 (scan_shard_reduce_publish: total -> every rank's slot array)
    is enqueued before any pass 2 (scan_shard_scan_peers: carry from its own
    slots), in one stream, so the in-kernel waits find their slots filled.  The
    slot arrays are G separate device buffers and peers = their device
    addresses, exactly what symmetric memory provides across GPUs."""
    import torch
    words = cuda.peer_slots_bytes(G) // 8
    slots = [torch.zeros(words, dtype=torch.int64, device="cuda") for _ in range(G)]
    peers = torch.tensor([s.data_ptr() for s in slots], dtype=torch.int64, device="cuda")
    wss = [cuda.shard_workspace(x) for x in x_shards]
    results = []
    for ep in epochs:
        for r in range(G):
            cuda.shard_reduce_publish(x_shards[r], peers.data_ptr(), G, r, ep, ws=wss[r])
        ys = [cuda.shard_scan_peers(x_shards[r], exclusive, slots[r], G, r, ep, ws=wss[r]) for r in range(G)]
        torch.cuda.synchronize()
        results.append([y.cpu().numpy() for y in ys])
    return results


@pytest.mark.parametrize("G", [1, 3, 8])
def test_peer_exchange_emulated_int8(cuda, oracle, inputs_mod, G):
    """Device-initiated totals exchange, int8 flags -> int32 exclusive, bit-exact
    against the oracle over the whole array; epochs 1, 2 and 65 / 66 (the slot
    ring of 64 wraps onto entries written by epochs 1 / 2)."""
    import torch
    from paper_2505_15112_b200.dist import shard_bounds
    n = G * 3 * 131072 + 12345
    x = inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n)
    ref = oracle.exclusive(x, "i8")
    bounds = [shard_bounds(n, G, r) for r in range(G)]
    shards = [torch.from_numpy(x[lo:hi]).cuda() for lo, hi in bounds]
    for ys in _emulated_peer_exchange(cuda, shards, True, G, (1, 2, 65, 66)):
        assert np.array_equal(np.concatenate(ys), ref)


def test_peer_exchange_emulated_fp32_edge_shards(cuda, oracle, inputs_mod):
    """fp32 inclusive with shards that take every pass-2 path: several blocks +
    a tail, shorter than one block (carry by the one-warp slot reader), an empty
    shard (publishes 0), and an unaligned shard (1-D fallback)."""
    import torch
    sizes = [3 * 131072 + 5, 1000, 0, 2 * 131072 + 3, 131072]
    n = sum(sizes)
    x = inputs_mod.fill_host(inputs_mod.F32_NORMAL, 4, 0, n + 1)
    y64, a64, _ = oracle.inclusive(x[:n], "f32")
    xd_all = torch.from_numpy(x).cuda()
    shards, lo = [], 0
    for i, m in enumerate(sizes):
        if i == 3:  # unaligned: a copy placed one element past an aligned start
            buf = torch.empty(m + 1, dtype=torch.float32, device="cuda")
            buf[1:].copy_(xd_all[lo:lo + m])
            shards.append(buf[1:])
        else:
            shards.append(xd_all[lo:lo + m].clone())
        lo += m
    for ys in _emulated_peer_exchange(cuda, shards, False, len(sizes), (7, 8)):
        got = np.concatenate(ys)
        bad, worst, at = oracle.check_f32(got, y64, a64)
        assert bad == 0, (worst, at)
