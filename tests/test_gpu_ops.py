"""GPU parity of the scan-based operators (include/scan_ops.h) against the CPU
oracle (oracle/oracle_ops.c): split / compress (P281-285) and the LSB radix
sort by per-bit splits (P286-287).  All results are integer / byte moves, so
every comparison is bit-exact.  Sizes span several 8192-element tiles and
ragged tails; edge cases: empty, 1 element, unaligned buffers, all-true /
all-false masks, nonzero flags other than 1 (R12), NaN / inf / signed zeros.
At full size (the C3 mask, n = 2^30) the outputs are checked by properties
that pin a split completely."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SIZES = [1, 15, 16, 17, 8191, 8192, 8193, 3 * 8192 + 5, 100003, (1 << 20) + 3]
PAYLOAD = {1: torch.int8, 2: torch.float16, 4: torch.int32, 8: torch.int64}


def _flags(inputs_mod, n, seed):
    return inputs_mod.fill_host(inputs_mod.I8_FLAG, seed, 0, n)


def _payload(n, es, seed):
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 256, n * es, dtype=np.uint8)
    return torch.from_numpy(raw).view(PAYLOAD[es]).cuda(), raw.view({1: np.int8, 2: np.uint16, 4: np.int32, 8: np.int64}[es])


@pytest.mark.parametrize("es", [1, 2, 4, 8])
@pytest.mark.parametrize("compress", [False, True])
@pytest.mark.parametrize("kernel", ["default", "warp", "direct", "block"])
def test_split_sizes(cuda, oracle, inputs_mod, monkeypatch, es, compress, kernel):
    if kernel != "default":  # every scatter kernel, whichever the default picks
        monkeypatch.setenv("SCAN_SPLIT_WARP", "0" if kernel == "block" else "1")
    if kernel == "direct":  # the warp kernel with direct element stores instead of staged runs
        monkeypatch.setenv("SCAN_SPLIT_DIRECT", "1")
    for n in SIZES:
        f = _flags(inputs_mod, n, seed=n)
        xd, xh = _payload(n, es, seed=n + es)
        z, idx, cnt = cuda.split(xd, torch.from_numpy(f).cuda(), compress=compress)
        zr, ir, T = oracle.split(xh, f, compress=compress)
        assert int(cnt.item()) == T
        m = T if compress else n
        got = z[:m].cpu().numpy().view(xh.dtype)
        assert np.array_equal(got, zr), (n, es)
        assert np.array_equal(idx[:m].cpu().numpy(), ir), (n, es)


def test_split_edge_cases(cuda, oracle):
    dev = torch.device("cuda")
    # empty
    z, idx, cnt = cuda.split(torch.empty(0, dtype=torch.int32, device=dev), torch.empty(0, dtype=torch.int8, device=dev))
    assert z.numel() == 0 and int(cnt.item()) == 0
    n = 3 * 8192 + 7
    x = np.arange(n, dtype=np.int32)
    for f in (np.ones(n, np.int8), np.zeros(n, np.int8),
              np.random.default_rng(1).choice(np.array([0, 1, -3, 2, 127, -128], np.int8), n)):
        z, idx, cnt = cuda.split(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda())
        zr, ir, T = oracle.split(x, f)
        assert int(cnt.item()) == T
        assert np.array_equal(z.cpu().numpy(), zr) and np.array_equal(idx.cpu().numpy(), ir)


def test_split_unaligned(cuda, oracle, inputs_mod):
    n = 50001
    f = _flags(inputs_mod, n + 3, seed=7)
    xd, xh = _payload(n + 3, 2, seed=8)
    fd = torch.from_numpy(f).cuda()
    for off in (1, 3):
        z, idx, cnt = cuda.split(xd[off:off + n], fd[off:off + n])
        zr, ir, T = oracle.split(xh[off:off + n].copy(), f[off:off + n].copy())
        assert int(cnt.item()) == T
        assert np.array_equal(z.cpu().numpy().view(np.uint16), zr) and np.array_equal(idx.cpu().numpy(), ir)


@pytest.mark.parametrize("es", [1, 2])
@pytest.mark.parametrize("kernel", ["staged", "single_pass", "direct"])
def test_compress_no_indices(cuda, oracle, inputs_mod, monkeypatch, es, kernel):
    """compress without indices: the two-pass staged-run kernel (default; 16-byte
    stores from a per-warp run aligned to the destination), the single-pass
    look-back kernel (A/B) and the direct-store kernel, on the recipe's mask and
    on all-true / all-false / sparse / alternating masks."""
    if kernel == "direct":
        monkeypatch.setenv("SCAN_SPLIT_DIRECT", "1")
    if kernel == "single_pass":
        monkeypatch.setenv("SCAN_COMPRESS_SP", "1")
    for n in SIZES + [3 * 4096 + 17, 8192 * 5, 148 * 65536 * 2 + 12345]:
        xd, xh = _payload(n, es, seed=n + 11 * es)
        rng = np.random.default_rng(n)
        masks = [_flags(inputs_mod, n, seed=n + 1), np.ones(n, np.int8), np.zeros(n, np.int8),
                 (rng.random(n) < 0.01).astype(np.int8), (np.arange(n) % 2).astype(np.int8)]
        for f in masks:
            z, _, cnt = cuda.split(xd, torch.from_numpy(f).cuda(), compress=True, with_idx=False)
            zr, _, T = oracle.split(xh, f, compress=True)
            assert int(cnt.item()) == T
            assert np.array_equal(z[:T].cpu().numpy().view(xh.dtype), zr), (n, es, int(f.sum()))


def test_compress_matches_masked_select(cuda, inputs_mod):
    n = 1 << 20
    f = torch.from_numpy(_flags(inputs_mod, n, seed=2)).cuda()
    x = torch.randn(n, device="cuda")
    got = cuda.compress(x, f)
    assert torch.equal(got, torch.masked_select(x, f != 0))


@pytest.mark.slow
def test_split_full_size_properties(cuda, inputs_mod):
    """C3's mask (n = 2^30, Bernoulli(0.5), seed 2) with an int16 payload: the
    count equals the popcount, idx is the stable partition (trues ascending,
    then falses ascending) and z = x[idx] -- which determines the split."""
    n = 1 << 30
    f = torch.empty(n, dtype=torch.int8, device="cuda")
    inputs_mod.fill_device(inputs_mod.I8_FLAG, 2, 0, n, 0, f)
    x = torch.arange(n, device="cuda", dtype=torch.int32).to(torch.int16)
    z, idx, cnt = cuda.split(x, f)
    T = int(cnt.item())
    assert T == int(f.sum(dtype=torch.int64).item())
    assert abs(T - n // 2) < 6 * (n ** 0.5) / 2
    idx64 = idx.to(torch.int64)
    assert bool((f[idx64[:T]] != 0).all()) and bool((f[idx64[T:]] == 0).all())
    assert bool((idx64[1:T] > idx64[:T - 1]).all()) and bool((idx64[T + 1:] > idx64[T:-1]).all())
    assert torch.equal(z, x[idx64])


# ----------------------------------------------------------------- radix sort
KEY_NP = {torch.float16: (np.float16, "f16"), torch.int16: (np.int16, "i16"),
          torch.int32: (np.int32, "i32"), torch.float32: (np.float32, "f32")}


def _keys(dt, n, seed):
    rng = np.random.default_rng(seed)
    npdt, _ = KEY_NP[dt]
    if dt in (torch.float16, torch.float32):
        k = (rng.standard_normal(n) * 50).astype(npdt)
        specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 1.0, -1.0], npdt)
        k[rng.integers(0, n, min(n, 64))] = rng.choice(specials, min(n, 64))
    else:
        info = np.iinfo(npdt)
        k = rng.integers(info.min, info.max, n, endpoint=True).astype(npdt)
    if n > 10:
        k[::9] = k[5]  # ties: stability
    return k


@pytest.mark.parametrize("dt", [torch.float16, torch.int16, torch.int32, torch.float32])
@pytest.mark.parametrize("desc", [False, True])
def test_radix_sort_parity(cuda, oracle, dt, desc):
    sizes = [1, 17, 8193, 100003] if dt in (torch.int32, torch.float32) else [1, 17, 8193, 100003, (1 << 18) + 9]
    for n in sizes:
        k = _keys(dt, n, seed=n)
        kd = torch.from_numpy(k).cuda()
        out, idx = cuda.radix_sort(kd, descending=desc)
        ro, ri = oracle.radix_sort(k, KEY_NP[dt][1], descending=desc)
        bits = np.uint16 if k.itemsize == 2 else np.uint32
        assert np.array_equal(idx.cpu().numpy(), ri), (dt, n)
        assert np.array_equal(out.cpu().numpy().view(bits), ro.view(bits)), (dt, n)


@pytest.mark.parametrize("n", [1 << 20, 1 << 24])  # 2^24 = bench_ops' sort workload
def test_radix_sort_matches_torch_sort_stable(cuda, n):
    """Against torch.sort(stable=True) (CUB) on NaN-free keys without -0."""
    for dt in (torch.float16, torch.float32, torch.int32):
        k = (torch.randn(n, device="cuda") * 1000).to(dt)
        if dt.is_floating_point:
            k[k == 0] = 1
        for desc in (False, True):
            out, idx = cuda.radix_sort(k, descending=desc)
            ref, ridx = torch.sort(k, stable=True, descending=desc)
            assert torch.equal(out, ref) and torch.equal(idx.to(torch.int64), ridx)


@pytest.mark.parametrize("dt", [torch.float16, torch.int16, torch.int32, torch.float32])
@pytest.mark.parametrize("desc", [False, True])
def test_radix_sort_rows_parity(cuda, oracle, dt, desc):
    """The row-batched sort (scan_radix_sort_rows): every row equals the
    oracle's 1-bit-split sort of that row (keys and column indices), for rows of
    one tile, several tiles + a ragged tile, and column counts that are not a
    multiple of 4 (the non-ring tile path)."""
    for R, C in ((1, 1), (5, 17), (3, 8192), (4, 8193), (7, 3 * 8192 + 5), (2, 100003), (64, 1000)):
        k = _keys(dt, R * C, seed=R * 31 + C).reshape(R, C)
        out, idx = cuda.radix_sort_rows(torch.from_numpy(k).cuda(), descending=desc)
        out, idx = out.cpu().numpy(), idx.cpu().numpy()
        bits = np.uint16 if k.itemsize == 2 else np.uint32
        for r in range(R):
            ro, ri = oracle.radix_sort(k[r], KEY_NP[dt][1], descending=desc)
            assert np.array_equal(idx[r], ri), (dt, R, C, r)
            assert np.array_equal(out[r].view(bits), ro.view(bits)), (dt, R, C, r)


def test_radix_sort_rows_matches_torch_sort_c4(cuda, inputs_mod):
    """C4 softmax rows (the top-p sort path's input), descending stable: equals
    torch.sort(descending=True, stable=True) row by row (keys and indices)."""
    R, C = 512, 131072
    P = torch.empty((R, C), dtype=torch.float32, device="cuda")
    inputs_mod.fill_device(inputs_mod.F32_SOFTMAX, 3, 0, R, C, P)
    out, idx = cuda.radix_sort_rows(P, descending=True)
    ref, ridx = torch.sort(P, dim=1, descending=True, stable=True)
    assert torch.equal(out, ref) and torch.equal(idx.to(torch.int64), ridx)


# ---------------------------------------------------------- sampling (P463, P299)
def _valid_interval(S64, j, t, tol):
    """j is a valid inverse-transform draw for threshold t on the fp64 prefix
    sums S64 (within the scan tolerance tol): S_{j-1} <= t < S_j."""
    lo = S64[j - 1] if j > 0 else 0.0
    return lo <= t + tol and S64[j] > t - tol


def test_weighted_sample_parity(cuda, oracle, inputs_mod):
    rng = np.random.default_rng(21)
    for n in (1, 17, 8193, 100003, 1 << 20):
        w = rng.random(n).astype(np.float32)
        w[rng.random(n) < 0.1] = 0
        if w.sum() == 0:
            w[0] = 1
        wd = torch.from_numpy(w).cuda()
        S64 = np.cumsum(w.astype(np.float64))
        tol = 1e-6 * S64[-1] + 1e-6
        same = 0
        thetas = [0.0, 0.5, 0.999, *rng.random(5)]
        for th in thetas:
            got = int(cuda.weighted_sample(wd, th).item())
            ref = oracle.weighted_sample(w, th)
            assert 0 <= got < n and w[got] > 0
            assert _valid_interval(S64, got, th * S64[-1], tol), (n, th, got, ref)
            same += got == ref
        assert same >= len(thetas) - 1  # differs only when t sits within rounding of a boundary


@pytest.mark.parametrize("method", ["select", "sort"])
def test_top_p_parity(cuda, oracle, inputs_mod, method):
    """C4-style rows (softmax(4 z)), several p; token and nucleus size match the
    oracle except where a threshold sits within float rounding of a boundary,
    and are always valid draws within the scan tolerance."""
    R, C = 64, 131072
    P = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 0, R, C)
    Pd = torch.from_numpy(P).cuda()
    rng = np.random.default_rng(3)
    u = rng.random(R).astype(np.float32)
    ud = torch.from_numpy(u).cuda()
    for p in (0.0, 0.5, 0.9, 0.95, 2.0):
        tok, kept = cuda.top_p_sample(Pd, p, ud, method=method)
        tok, kept = tok.cpu().numpy(), kept.cpu().numpy()
        agree = 0
        for r in range(R):
            rt, rk = oracle.top_p_sample(P[r], float(np.float32(p)), float(u[r]))  # p as the C ABI's fp32
            order = np.argsort(-P[r].astype(np.float64), kind="stable")
            C64 = np.cumsum(P[r][order].astype(np.float64))
            tol = 1e-6 * C64[-1] + 1e-6
            K = int(kept[r])
            # nucleus: smallest prefix with mass >= p (R15), within tolerance
            assert K >= 1 and (K == C or C64[K - 1] >= p - tol)
            assert K == 1 or C64[K - 2] < p + tol
            rank = int(np.nonzero(order == tok[r])[0][0])
            assert rank < K and _valid_interval(C64, rank, float(u[r]) * C64[K - 1], tol)
            agree += (tok[r] == rt) and (K == rk)
        assert agree >= R - 2, (p, agree)


def test_top_p_select_edge_rows(cuda, oracle):
    """Sort-free top-p on hand-made rows: ties across the nucleus boundary
    (stable index order), a flat row that needs the sort fallback, zeros, a
    single dominant token, a ragged column count, a level of more than 2048 keys
    (full candidate sort), many levels with ties in each (the draw's level ahead
    of the nucleus level), a superset above 8192 candidates (re-read fallback)."""
    C = 50001
    rows = []
    r0 = np.zeros(C, np.float32); r0[[5, 17, 900, 40000]] = 0.25; rows.append(r0)     # 4-way tie
    r1 = np.full(C, 1.0 / C, np.float32); rows.append(r1)                             # flat: fallback
    r2 = np.zeros(C, np.float32); r2[123] = 1.0; rows.append(r2)                      # one token
    rng = np.random.default_rng(4)
    r3 = rng.random(C).astype(np.float32) ** 8; r3 /= r3.sum(); rows.append(r3)
    r4 = np.zeros(C, np.float32); r4[rng.choice(C, 3000, replace=False)] = 1.0 / 3000; rows.append(r4)  # level > 2048
    r5 = np.zeros(C, np.float32)                                                       # many levels, ties in each
    for k in range(12):
        r5[rng.choice(C, 40, replace=False)] += np.float32(2.0 ** -(k / 3.0))
    r5 /= r5.sum(); rows.append(r5)
    r6 = np.zeros(C, np.float32); r6[:10000] = 1e-4; rows.append(r6)                  # superset > 8192
    P = np.stack(rows)
    u = np.array([0.1, 0.5, 0.9, 0.77, 0.3, 0.999, 0.6], np.float32)
    for p in (0.05, 0.3, 0.6, 0.9, 0.999):
        tok, kept = cuda.top_p_sample(torch.from_numpy(P).cuda(), p, torch.from_numpy(u).cuda())
        for r in range(len(rows)):
            # the C ABI takes p as fp32: the oracle gets the same value
            p32 = float(np.float32(p))
            rt, rk = oracle.top_p_sample(P[r], p32, float(u[r]))
            if r in (1, 6):
                # more than 8192 candidates: the sort-path fallback (torch.sort + the fp32 row
                # scan), exact only up to the scan tolerance -- check validity there
                order = np.argsort(-P[r].astype(np.float64), kind="stable")
                C64 = np.cumsum(P[r][order].astype(np.float64))
                tol = 1e-6 * C64[-1] + 1e-6
                K = int(kept[r])
                assert K >= 1 and (K == C or C64[K - 1] >= p32 - tol) and (K == 1 or C64[K - 2] < p32 + tol)
                rank = int(np.nonzero(order == int(tok[r]))[0][0])
                assert rank < K and _valid_interval(C64, rank, float(u[r]) * C64[K - 1], tol), (p, r)
            else:
                assert int(tok[r]) == rt and int(kept[r]) == rk, (p, r, int(tok[r]), rt, int(kept[r]), rk)


def test_top_p_select_retry_paths(cuda, oracle, inputs_mod, monkeypatch):
    """The select kernel's retries: (a) a row whose running-maximum superset
    overflows (the early maximum is tiny) but whose final-maximum window fits;
    (b) a row whose nucleus reaches 12.6 octaves below the maximum, past the
    first attempt's 12.25-octave window (redone from the fixed-threshold
    attempt); (c) C4 rows with a 5-octave first window, so most rows are redone.
    Every token and nucleus size is the oracle's."""
    C = 131072
    rng = np.random.default_rng(11)
    M = np.float32(0.01)
    ra = np.zeros(C, np.float32)
    ra[:2048] = 1e-12                                                        # tiny early maximum
    ra[2048:22048] = M * np.float32(2.0 ** -15)                               # below the final window
    hot = rng.choice(np.arange(30000, C), 3000, replace=False)
    ra[hot] = M * (0.5 + 0.5 * rng.random(3000)).astype(np.float32)
    rb = np.zeros(C, np.float32)
    rb[77] = M
    far = rng.choice(np.arange(1000, C), 5000, replace=False)
    rb[far] = M * np.float32(2.0 ** -12.6)                                    # 12.6 octaves down
    P = np.stack([ra, rb])
    u = np.array([0.35, 0.8], np.float32)
    for p in (0.5, 0.9, 0.99):
        tok, kept = cuda.top_p_sample(torch.from_numpy(P).cuda(), p, torch.from_numpy(u).cuda())
        for r in range(2):
            rt, rk = oracle.top_p_sample(P[r], float(np.float32(p)), float(u[r]))
            assert int(tok[r]) == rt and int(kept[r]) == rk, (p, r, int(tok[r]), rt, int(kept[r]), rk)
    # (c) forced redo of most C4 rows (the window knob is read at every launch)
    R = 16
    Pc = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 0, R, C)
    uc = rng.random(R).astype(np.float32)
    monkeypatch.setenv("SCAN_TOPP_W0", "40")
    tok, kept = cuda.top_p_sample(torch.from_numpy(Pc).cuda(), 0.9, torch.from_numpy(uc).cuda())
    monkeypatch.delenv("SCAN_TOPP_W0")
    for r in range(R):
        rt, rk = oracle.top_p_sample(Pc[r], float(np.float32(0.9)), float(uc[r]))
        assert int(tok[r]) == rt and int(kept[r]) == rk, (r, int(tok[r]), rt, int(kept[r]), rk)


@pytest.mark.slow
def test_top_p_full_c4(cuda, oracle, inputs_mod):
    """bench_ops' top-p workload (4096 C4 rows, p = 0.9): the sort-free path and
    the sort path agree on every row; a sample of rows matches the oracle."""
    R, C = 4096, 131072
    P = torch.empty((R, C), dtype=torch.float32, device="cuda")
    inputs_mod.fill_device(inputs_mod.F32_SOFTMAX, 3, 0, R, C, P)
    u = torch.rand(R, generator=torch.Generator(device="cuda").manual_seed(7), device="cuda")
    t1, k1 = cuda.top_p_sample(P, 0.9, u, method="select")
    t2, k2 = cuda.top_p_sample(P, 0.9, u, method="sort")
    # the sort path decides the nucleus on the fp32 row scan, the select path in
    # fp64 (the oracle's precision): K may differ where C_j sits within fp32
    # rounding of p; the drawn tokens agree
    assert int((t1 != t2).sum()) <= 2 and int((k1 != k2).sum()) <= 16
    uh = u.cpu().numpy()
    for r in range(0, R, 256):
        Ph = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, r, 1, C)[0]
        rt, rk = oracle.top_p_sample(Ph, 0.9, float(uh[r]))
        assert int(t1[r]) == rt and int(k1[r]) == rk, (r, int(t1[r]), rt, int(k1[r]), rk)
