"""Parity of the CUDA scan (through the C ABI) against the CPU oracle.

Integers: bit-exact.  Floats: the north_star tolerance
|gpu - oracle_fp64| <= 1e-6 * sum_{j<=i}|x_j| + 1e-6, element by element.
Sizes span several tiles (8192 elements) and ragged tails; edge cases cover
empty, 1 element, unaligned pointers, in-place, carry-in, strided rows.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

M32 = (1 << 32) - 1
TORCH_IN = {"i32": torch.int32, "f32": torch.float32, "f16": torch.float16, "i8": torch.int8}
NP_IN = {"i32": np.int32, "f32": np.float32, "f16": np.uint16, "i8": np.int8}


def host_input(inputs_mod, dt, n, seed=123, kind=None):
    if kind is None:
        kind = {"i32": inputs_mod.I32_FULL, "f32": inputs_mod.F32_NORMAL,
                "f16": inputs_mod.F16_NORMAL, "i8": inputs_mod.I8_FULL}[dt]
    return inputs_mod.fill_host(kind, seed, 0, n)


def to_dev(x, dt):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dt == "f16":
        t = t.view(torch.float16)
    return t.cuda()


def oracle_1d(oracle, x, dt, exclusive, carry=None):
    fn = oracle.exclusive if exclusive else oracle.inclusive
    return fn(x, dt, carry_in=carry)


def assert_parity(oracle, got, ref, dt):
    got = got.cpu().numpy().reshape(-1)
    if dt in ("i32", "i8"):
        assert got.dtype == np.int32
        bad = np.nonzero(got != ref.reshape(-1))[0]
        assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: {got[bad[:5]]} vs {ref.reshape(-1)[bad[:5]]}"
    else:
        y64, a64, _ = ref
        bad, worst, at = oracle.check_f32(got, y64, a64)
        assert bad == 0, f"{bad} elements out of tolerance; worst err/tol {worst} at {at}"
        return worst


SIZES = [1, 2, 3, 31, 32, 33, 127, 128, 129, 4095, 4096, 4097, 8191, 8192, 8193,
         3 * 8192 + 5, 65536, 65537, 100003, 1 << 20, (1 << 20) + 3]


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_1d_sizes(cuda, oracle, inputs_mod, dt, exclusive):
    for n in SIZES:
        x = host_input(inputs_mod, dt, n, seed=n)
        fn = cuda.exclusive if exclusive else cuda.inclusive
        got = fn(to_dev(x, dt))
        torch.cuda.synchronize()
        assert_parity(oracle, got, oracle_1d(oracle, x, dt, exclusive), dt)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_random_sizes_and_carry(cuda, oracle, inputs_mod, dt):
    rng = np.random.default_rng(7)
    for trial in range(6):
        n = int(rng.integers(1, 1 << 22))
        x = host_input(inputs_mod, dt, n, seed=trial)
        exclusive = bool(trial % 2)
        if dt in ("i32", "i8"):
            c = int(rng.integers(-(1 << 40), 1 << 40))
            carry = torch.tensor([c], dtype=torch.int64, device="cuda")
        else:
            c = float(rng.normal() * 1000)
            carry = torch.tensor([c], dtype=torch.float64, device="cuda")
        fn = cuda.exclusive if exclusive else cuda.inclusive
        got = fn(to_dev(x, dt), carry_in=carry)
        torch.cuda.synchronize()
        assert_parity(oracle, got, oracle_1d(oracle, x, dt, exclusive, carry=c), dt)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_unaligned(cuda, oracle, inputs_mod, dt):
    n = 50000
    for off_in in (0, 1, 2, 3):
        for off_out in (0, 1, 3):
            if off_in == 0 and off_out == 0:
                continue
            x = host_input(inputs_mod, dt, n + off_in, seed=off_in)
            xd = to_dev(x, dt)[off_in:]
            outb = torch.empty(n + off_out, dtype=torch.int32 if dt in ("i32", "i8")
                               else torch.float32, device="cuda")
            out = outb[off_out:]
            cuda.inclusive(xd, out=out)
            torch.cuda.synchronize()
            assert_parity(oracle, out, oracle_1d(oracle, x[off_in:], dt, False), dt)


@pytest.mark.parametrize("dt", ["i32", "f32"])
def test_in_place(cuda, oracle, inputs_mod, dt):
    n = 300007
    x = host_input(inputs_mod, dt, n)
    xd = to_dev(x, dt)
    cuda.inclusive(xd, out=xd)
    torch.cuda.synchronize()
    assert_parity(oracle, xd, oracle_1d(oracle, x, dt, False), dt)


@pytest.mark.parametrize("n", [4096, 65536, 100000])
def test_dependent_small_scans_pdl(cuda, oracle, inputs_mod, n):
    """Small scans are launched with programmatic dependent launch: a scan that
    reads the previous scan's output must still see all of it (the kernel waits
    on griddepcontrol before its first global access).  Chains of dependent
    scans, eagerly and replayed from a CUDA graph, against the oracle."""
    x = host_input(inputs_mod, "i32", n, seed=n)
    ref = x.copy()
    for _ in range(3):
        ref = oracle.inclusive(ref, "i32")
    xd = to_dev(x, "i32")
    a = torch.empty_like(xd)
    b = torch.empty_like(xd)
    c = torch.empty_like(xd)

    def chain():
        cuda.inclusive(xd, out=a)
        cuda.inclusive(a, out=b)
        cuda.inclusive(b, out=c)

    chain()
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), ref)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        chain()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(4):
                chain()
    for _ in range(3):
        c.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy(), ref)


def test_empty_and_errors(cuda):
    L = cuda.load()
    x = torch.empty(0, dtype=torch.int32, device="cuda")
    assert cuda.inclusive(x).numel() == 0
    # bad arguments are rejected without launching
    assert L.scan_inclusive(None, None, 10, 0, None, None, 0, None) == 1
    assert L.scan_inclusive(None, None, -1, 0, None, None, 0, None) == 1
    y = torch.zeros(100000, dtype=torch.int32, device="cuda")
    z = torch.zeros(100000, dtype=torch.int32, device="cuda")
    import ctypes
    assert L.scan_inclusive(ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                            100000, 7, None, None, 0, None) == 1           # bad dtype
    assert L.scan_inclusive(ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                            100000, 0, None, None, 0, None) == 2           # no workspace
    assert L.scan_inclusive(ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(y.data_ptr() + 4),
                            1000, 0, None, None, 0, None) == 1             # partial overlap


def test_repeat_calls_reuse_workspace(cuda, oracle, inputs_mod):
    """Epoch-tagged descriptors: 200 back-to-back calls on one workspace with
    varying sizes must all be exact (no stale descriptor is ever read)."""
    rng = np.random.default_rng(3)
    xs = host_input(inputs_mod, "i32", 1 << 20, seed=99)
    xd = to_dev(xs, "i32")
    ref = oracle.inclusive(xs, "i32")
    outs = []
    for i in range(200):
        n = int(rng.integers(8193, 1 << 20))
        outs.append((n, cuda.inclusive(xd[:n])))
    torch.cuda.synchronize()
    for n, o in outs:
        assert np.array_equal(o.cpu().numpy(), ref[:n])


def test_float_bitwise_repeatable_c2_like(cuda, inputs_mod):
    """fp16 U[0,1) (C2-like): fp64 carries are exact, so repeated runs give identical bits."""
    n = 1 << 24
    x = to_dev(inputs_mod.fill_host(inputs_mod.F16_U01, 1, 0, n), "f16")
    a = cuda.inclusive(x)
    b = cuda.inclusive(x)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


# ------------------------------------------------------------------ rows

@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_rows(cuda, oracle, inputs_mod, dt):
    for R, C in ((1, 1), (7, 3), (5, 31), (148, 32), (7, 1000), (3, 4096), (5, 8192), (4, 8193),
                 (9, 65536), (2, 131072), (300, 513)):
        x = host_input(inputs_mod, dt, R * C, seed=R * 1000 + C).reshape(R, C)
        for exc in (False, True):
            got = cuda.rows(to_dev(x, dt), exclusive=exc)
            torch.cuda.synchronize()
            if dt in ("i32", "i8"):
                ref = np.stack([oracle_1d(oracle, x[r], dt, exc) for r in range(R)])
                assert_parity(oracle, got, ref, dt)
            else:
                parts = [oracle_1d(oracle, x[r], dt, exc) for r in range(R)]
                ref = tuple(np.concatenate([p[k] for p in parts]) for k in range(3))
                assert_parity(oracle, got, ref, dt)


@pytest.mark.parametrize("dt", ["i32", "f32"])
def test_rows_strided(cuda, oracle, inputs_mod, dt):
    R, C, S = 6, 20000, 20004
    x = host_input(inputs_mod, dt, R * S).reshape(R, S)
    xd = to_dev(x, dt)[:, :C]
    outb = torch.empty((R, C + 8), dtype=torch.int32 if dt == "i32" else torch.float32,
                       device="cuda")
    out = outb[:, 3:3 + C]
    cuda.rows(xd, out=out)
    torch.cuda.synchronize()
    for r in range(R):
        assert_parity(oracle, out[r], oracle_1d(oracle, np.ascontiguousarray(x[r, :C]), dt, False),
                      dt)


def test_rows_exhaustive_12bit_flags(cuda, oracle):
    """All 4096 length-12 0/1 flag patterns in one scan_rows call."""
    pats = np.arange(4096)
    X = ((pats[:, None] >> np.arange(12)[None, :]) & 1).astype(np.int8)
    got = cuda.rows(to_dev(X, "i8")).cpu().numpy()
    want = np.stack([oracle.inclusive(X[p], "i8") for p in range(4096)])
    assert np.array_equal(got, want)
    got = cuda.rows(to_dev(X, "i8"), exclusive=True).cpu().numpy()
    want = np.stack([oracle.exclusive(X[p], "i8") for p in range(4096)])
    assert np.array_equal(got, want)


# ------------------------------------------------------------ total / carry

@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_total_and_carry(cuda, oracle, inputs_mod, dt):
    for n in (1, 1000, 8193, 1 << 20, 12345677):
        x = host_input(inputs_mod, dt, n, seed=n)
        t = cuda.total(to_dev(x, dt))
        torch.cuda.synchronize()
        ref = oracle.total(x, dt)
        if dt in ("i32", "i8"):
            assert int(t.item()) == ref
        else:
            absum = oracle.FloatScan(dt)(x, want64=False, want32=False)[1][-1]
            assert abs(t.item() - ref) <= 2 * n * 2.0 ** -53 * absum
        t2 = cuda.total(to_dev(x, dt))
        assert t2.item() == t.item()          # fixed summation order: identical bits
    G = 5
    cdt = torch.int64 if dt in ("i32", "i8") else torch.float64
    totals = torch.tensor([3, -7, 11, 100, 5], dtype=cdt, device="cuda")
    for r in range(G):
        c = cuda.carry_from_totals(totals, r, TORCH_IN[dt])
        assert c.item() == sum([3, -7, 11, 100, 5][:r])


# ---------------------------------------------- large 1-D (MCScan + L2 split)

LARGE = [(1 << 20) + 1, (1 << 20) + 17, (1 << 20) + 31, 3 * (1 << 20) + 5, (1 << 22) + 7,
         (1 << 24) + 13, 5 * (1 << 22) + 100003]


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_large_ragged(cuda, oracle, inputs_mod, dt):
    """Multi-chunk arrays whose length is not a multiple of the 128-byte TMA
    row, of the tile or of the chunk: exercises the chunk barrier, the block
    carries and the directly loaded/stored tail."""
    for i, n in enumerate(LARGE):
        x = host_input(inputs_mod, dt, n, seed=1000 + i)
        exclusive = bool(i % 2)
        carry = None
        c = None
        if i % 3 == 2:
            if dt in ("i32", "i8"):
                c = 123456789012
                carry = torch.tensor([c], dtype=torch.int64, device="cuda")
            else:
                c = -777.25
                carry = torch.tensor([c], dtype=torch.float64, device="cuda")
        fn = cuda.exclusive if exclusive else cuda.inclusive
        got = fn(to_dev(x, dt), carry_in=carry)
        torch.cuda.synchronize()
        assert_parity(oracle, got, oracle_1d(oracle, x, dt, exclusive, carry=c), dt)


@pytest.mark.parametrize("dt", ["i8", "f32", "i32", "f16"])
def test_sharded_emulation(cuda, oracle, inputs_mod, dt):
    """The multi-GPU Reduce-Scan-Scan path on one GPU: the array is split into
    G contiguous shards; per shard scan_total, an emulated all-gather
    (torch.cat), carry_from_totals and a scan with carry-in (the same
    dist.rss_scan host logic the NCCL path runs).  The concatenation must equal
    the oracle over the whole array (bit-exact for integers)."""
    from paper_2505_15112_b200.dist import rss_scan, shard_bounds
    n, G = 3 * (1 << 20) + 12345, 4
    x = host_input(inputs_mod, dt, n, seed=77)
    xd = to_dev(x, dt)
    exclusive = dt == "i8"
    shards = [xd[slice(*shard_bounds(n, G, r))] for r in range(G)]
    wss = [cuda.shard_workspace(s) for s in shards]  # one per "rank"
    totals_all = torch.cat([cuda.shard_reduce(s, ws=w) for s, w in zip(shards, wss)])
    ref_tot = torch.cat([cuda.total(s) for s in shards])
    if dt in ("i32", "i8"):
        assert torch.equal(totals_all, ref_tot)
    else:
        assert torch.allclose(totals_all, ref_tot, rtol=1e-12, atol=1e-9)
    outs = []
    for r, s in enumerate(shards):
        y, totals, carry = rss_scan(
            s, exclusive, r, G,
            local_total=lambda xl: totals_all[r:r + 1],
            all_gather=lambda t: totals_all,
            carry_of=lambda totals, rr: cuda.carry_from_totals(totals, rr, s.dtype),
            local_scan=lambda xl, exc, c: cuda.shard_scan(xl, exc, carry_in=c, ws=wss[r]))
        outs.append(y)
    got = torch.cat(outs)
    torch.cuda.synchronize()
    assert_parity(oracle, got, oracle_1d(oracle, x, dt, exclusive), dt)
    if dt in ("i32", "i8"):  # integers are unique: bit-exact against the single-GPU scan
        whole = (cuda.exclusive if exclusive else cuda.inclusive)(xd)
        assert torch.equal(got, whole)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_rows_many_tiles_strided(cuda, oracle, inputs_mod, dt):
    """Rows of several tiles with a ragged last tile and padded (16-byte
    aligned) row strides: the one-CTA-per-row kernel (rowscan.cuh)."""
    R = 13
    C = 40064 if dt == "i8" else 40000
    S = C + 128
    x = host_input(inputs_mod, dt, R * S, seed=4242).reshape(R, S)
    xd = to_dev(x, dt)[:, :C]
    out_b = torch.empty((R, C + 64), dtype=torch.int32 if dt in ("i32", "i8") else torch.float32,
                        device="cuda")
    for exc in (False, True):
        out = out_b[:, :C]
        cuda.rows(xd, exclusive=exc, out=out)
        torch.cuda.synchronize()
        for r in range(R):
            assert_parity(oracle, out[r], oracle_1d(oracle, np.ascontiguousarray(x[r, :C]), dt, exc), dt)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
def test_host_streaming(cuda, oracle, inputs_mod, dt):
    """scan_host: pinned host in -> chunked H2D / scan / D2H pipeline -> host out,
    with ragged chunk counts (carry chained across chunks on the device)."""
    n = 5 * (1 << 20) + 777
    x = host_input(inputs_mod, dt, n, seed=31)
    t = torch.from_numpy(x)
    if dt == "f16":
        t = t.view(torch.float16)
    h = t.pin_memory()
    for exc, chunk in ((False, 1 << 20), (True, 3 * (1 << 19) + 5), (False, n)):
        got = cuda.host_scan(h, exclusive=exc, chunk=chunk)
        torch.cuda.synchronize()
        assert_parity(oracle, got, oracle_1d(oracle, x, dt, exc), dt)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_shard_two_pass(cuda, oracle, inputs_mod, dt, exclusive):
    """scan_shard_reduce + scan_shard_scan (block rows of 131,072 + ragged tail,
    carry-in, unaligned fallback) == the oracle with the same carry."""
    carry_val = {"i32": 123456789, "i8": -77, "f32": 3.25, "f16": -1.5}[dt]
    cdt = torch.int64 if dt in ("i32", "i8") else torch.float64
    for n in (131072, 3 * 131072, 5 * 131072 + 777, 40000):
        x = host_input(inputs_mod, dt, n + 1, seed=n)
        for off in (0, 1):
            xs = np.ascontiguousarray(x[off:off + n])
            xd = to_dev(x, dt)[off:off + n]
            ws = cuda.shard_workspace(xd)
            tot = cuda.shard_reduce(xd, ws=ws)
            ref_tot = oracle.total(xs, dt)
            if dt in ("i32", "i8"):
                assert int(tot.item()) == ref_tot
            else:
                assert abs(float(tot.item()) - ref_tot) <= 1e-9 * max(1.0, abs(ref_tot))
            c = torch.tensor([carry_val], dtype=cdt, device="cuda")
            got = cuda.shard_scan(xd, exclusive, carry_in=c, ws=ws)
            assert_parity(oracle, got, oracle_1d(oracle, xs, dt, exclusive, carry=carry_val), dt)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_rows_tiny_contiguous(cuda, oracle, inputs_mod, dt, exclusive):
    """Contiguous rows of <= 32 columns take the shared-memory tile kernel
    (k_rows_tile: 16-byte staged loads / stores, a thread per row); ragged last
    tile (rows not a multiple of 256) and a ragged vector tail."""
    for R, C in [(1, 1), (1000, 1), (777, 3), (513, 17), (300, 32), (256 * 3 + 5, 31)]:
        x = host_input(inputs_mod, dt, R * C, seed=R * 13 + C).reshape(R, C)
        got = cuda.rows(to_dev(x, dt), exclusive=exclusive)
        torch.cuda.synchronize()
        if dt in ("i32", "i8"):
            assert np.array_equal(got.cpu().numpy(), oracle.rows(x, dt, exclusive=exclusive)), (R, C)
        else:
            y64, a64, _ = oracle.rows(x, dt, exclusive=exclusive)
            bad, worst, at = oracle.check_f32(got.cpu().numpy(), y64, a64)
            assert bad == 0, (R, C, worst, at)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_rows_tiny_strided(cuda, oracle, inputs_mod, dt, exclusive):
    """Strided rows of <= 32 columns, every row start 16-byte aligned in and out
    (the staged tile kernel's strided addressing) and not (the shuffle kernel):
    ragged row counts, input and output strides both wider than the row."""
    es = {"i32": 4, "f32": 4, "f16": 2, "i8": 1}[dt]
    for R, C, S_in, S_out in [(1000, 4, 8, 12), (777, 8, 24, 16), (513, 16, 48, 20), (300, 32, 64, 36),
                              (257, 32, 32 + 16 // es, 40), (999, 12, 16, 16), (65, 5, 8, 8)]:
        x = host_input(inputs_mod, dt, R * S_in, seed=R * 5 + C).reshape(R, S_in)
        xd = to_dev(x, dt)[:, :C]
        outb = torch.empty((R, S_out), dtype=torch.int32 if dt in ("i32", "i8") else torch.float32, device="cuda")
        out = outb[:, :C]
        cuda.rows(xd, exclusive=exclusive, out=out)
        torch.cuda.synchronize()
        xc = np.ascontiguousarray(x[:, :C])
        if dt in ("i32", "i8"):
            assert np.array_equal(out.cpu().numpy(), oracle.rows(xc, dt, exclusive=exclusive)), (R, C)
        else:
            y64, a64, _ = oracle.rows(xc, dt, exclusive=exclusive)
            bad, worst, at = oracle.check_f32(out.cpu().numpy(), y64, a64)
            assert bad == 0, (R, C, worst, at)


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_rows_short_and_few_long(cuda, oracle, inputs_mod, dt, exclusive):
    """Row shapes of every row path: tiny rows (segmented warp scan, several
    rows per warp), short rows (a warp per row), few long rows (one MCScan per
    row); strided rows for the first two."""
    shapes = [(1000, 1), (777, 3), (513, 17), (300, 32), (257, 33), (129, 1000), (65, 2048),
              (33, 4095), (9, 4096), (3, (1 << 22) + 5),
              (3, 1 << 19), (7, 12288 * 16), (2, 1 << 20), (150, 16384), (5, 300007), (40, 30011),
              (74, 16384), (74, 24576), (74, 14200), (20, 65537)]
    for R, C in shapes:
        S = C + (16 if C < 8192 else 0)
        x = host_input(inputs_mod, dt, R * S, seed=R * 7 + C).reshape(R, S)
        xd = to_dev(x, dt)[:, :C]
        got = cuda.rows(xd, exclusive=exclusive)
        torch.cuda.synchronize()
        xc = np.ascontiguousarray(x[:, :C])
        if dt in ("i32", "i8"):
            ref = oracle.rows(xc, dt, exclusive=exclusive)
            assert np.array_equal(got.cpu().numpy(), ref), (R, C)
        else:
            y64, a64, _ = oracle.rows(xc, dt, exclusive=exclusive)
            bad, worst, at = oracle.check_f32(got.cpu().numpy(), y64, a64)
            assert bad == 0, (R, C, worst, at)
