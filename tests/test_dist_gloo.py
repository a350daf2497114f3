"""Multi-rank host logic of the sharded scan (paper_2505_15112_b200.dist) on CPU:
world_size 2 (and 3) over gloo, with the per-rank operations bound to the
oracle.  Checks that the concatenation of the rank outputs equals the
unsharded scan (bit-exact for integers) and that the carry composition and
the all-gather order are right.  The CUDA bindings of the same function are
exercised on the GPU by tests/test_gpu_parity.py::test_sharded_emulation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, kind, dt, exclusive, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import inputs
        import oracle
        from paper_2505_15112_b200.dist import rss_scan, shard_bounds

        lo, hi = shard_bounds(n, world, rank)
        x = inputs.fill_host(kind, 5, lo, hi - lo)
        is_int = dt in ("i32", "i8")
        tdt = torch.int64 if is_int else torch.float64

        def local_total(xl):
            return torch.tensor([oracle.total(xl, dt)], dtype=tdt)

        def all_gather(t):
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return torch.cat(out)

        def carry_of(totals, r):
            c = totals[:r].sum() if r else torch.zeros((), dtype=tdt)
            return c.reshape(1)

        def local_scan(xl, exc, carry):
            c = carry.item()
            fn = oracle.exclusive if exc else oracle.inclusive
            y = fn(xl, dt, carry_in=int(c) if is_int else float(c))
            return y if is_int else y[0]          # fp64 values for the comparison

        y, totals, carry = rss_scan(x, exclusive, rank, world, local_total, all_gather, carry_of,
                                    local_scan)
        q.put((rank, lo, hi, np.asarray(y), totals.numpy(), carry.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,kind_name,dt,exclusive", [
    (2, 100003, "I8_FLAG", "i8", True),       # C3 shape, small
    (2, 65536, "I32_U100", "i32", False),
    (3, 50001, "I32_FULL", "i32", True),      # ragged shards, wrap-around
    (2, 40000, "F32_PM1", "f32", False),      # exact in fp64
])
def test_rss_gloo(world, n, kind_name, dt, exclusive, oracle, inputs_mod):
    kind = getattr(inputs_mod, kind_name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, kind, dt, exclusive, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = inputs_mod.fill_host(kind, 5, 0, n)
    whole = (oracle.exclusive if exclusive else oracle.inclusive)(x, dt)
    if dt == "f32":
        whole = whole[0]
    got = np.concatenate([r[3] for r in res])
    assert np.array_equal(got, whole)
    # every rank saw the same totals, in rank order, and carry_r = sum of lower totals
    totals = res[0][4]
    for r, lo, hi, _, t, c in res:
        assert np.array_equal(t, totals)
        assert c[0] == totals[:r].sum()
        assert totals[r] == oracle.total(x[lo:hi], dt)


def test_shard_bounds_cover():
    from paper_2505_15112_b200.dist import shard_bounds
    for n in (0, 1, 7, 100, 2 ** 32):
        for g in (1, 2, 3, 8):
            b = [shard_bounds(n, g, r) for r in range(g)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(g - 1))
            assert all(lo <= hi for lo, hi in b)
