"""Pins for the CPU oracle (tests run without a GPU).

Each test pins the oracle to something other than itself: a printed
example, a closed form, an invariant, brute force, an exact fixed-point
computation, or the paper's own matrix formulation of the scan (Eq. eqn:scan,
Alg. 1, Alg. 3) evaluated with numpy matmuls.  A plausible slip anywhere in
oracle_scan.c (dropped term, off-by-one, wrong sign, missing wrap, wrong
fp16 exponent bias, lost carry across chunks) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "scan_examples.json")
M32 = (1 << 32) - 1


def wrap32(v):
    """Python int -> int32 two's complement (R1)."""
    v &= M32
    return v - (1 << 32) if v >= (1 << 31) else v


def as_dt(x, dt):
    return np.asarray(x, dtype={"i32": np.int32, "i8": np.int8, "f32": np.float32}[dt])


# ---------------------------------------------------------------- golden

def test_golden_examples(oracle):
    data = json.load(open(GOLDEN))
    for case in data["cases"]:
        x = as_dt(case["x"], case["dt"])
        fn = oracle.inclusive if case["op"] == "inclusive" else oracle.exclusive
        got = fn(x, case["dt"])
        if case["dt"] == "f32":
            got = got[2]
        assert np.array_equal(np.asarray(got, dtype=np.float64),
                              np.asarray(case["y"], dtype=np.float64)), case["cite"]
    for case in data["rows"]:
        X = as_dt(case["X"], case["dt"])
        assert np.array_equal(oracle.rows(X, case["dt"]), np.asarray(case["Y"])), case["cite"]


# ---------------------------------------------------------- closed forms

@pytest.mark.parametrize("n", [0, 1, 2, 31, 1000, 65537])
def test_all_ones(oracle, n):
    """scan of all-ones = 1..n (north_star), exclusive = 0..n-1."""
    want_inc = np.arange(1, n + 1)
    want_exc = np.arange(0, n)
    for dt, one in (("i32", np.int32(1)), ("i8", np.int8(1))):
        x = np.full(n, one)
        assert np.array_equal(oracle.inclusive(x, dt), want_inc)
        assert np.array_equal(oracle.exclusive(x, dt), want_exc)
    x = np.ones(n, np.float32)
    y64, a64, y32 = oracle.inclusive(x, "f32")
    assert np.array_equal(y64, want_inc) and np.array_equal(y32, want_inc)
    assert np.array_equal(a64, want_inc)
    h = np.full(n, 0x3C00, np.uint16)          # fp16 1.0
    y64, a64, y32 = oracle.inclusive(h, "f16")
    assert np.array_equal(y64, want_inc)
    y64, _, _ = oracle.exclusive(x, "f32")
    assert np.array_equal(y64, want_exc)


def test_arithmetic_series_wraps(oracle):
    """x_i = a + d i  ->  y_i = (i+1) a + d i (i+1)/2  (mod 2^32), with overflow."""
    n = 100000
    a, d = 2_000_000_001, -7919
    i = np.arange(n, dtype=np.int64)
    x = ((a + d * i) & M32).astype(np.uint32).view(np.int32)
    y = oracle.inclusive(x, "i32")
    ii = [int(k) for k in range(n)]
    want = np.array([wrap32((k + 1) * a + d * k * (k + 1) // 2) for k in ii], dtype=np.int64)
    assert np.array_equal(y.astype(np.int64), want)


def test_alternating(oracle):
    n = 4097
    x = np.where(np.arange(n) % 2 == 0, 1, -1).astype(np.int32)
    y = oracle.inclusive(x, "i32")
    assert np.array_equal(y, (np.arange(n) % 2 == 0).astype(np.int32))
    y = oracle.inclusive(x.astype(np.int8), "i8")
    assert np.array_equal(y, (np.arange(n) % 2 == 0).astype(np.int32))


# ----------------------------------------------------------- brute force

@pytest.mark.parametrize("n", [1, 2, 3, 17, 256, 2048])
def test_bruteforce_int(oracle, inputs_mod, n):
    """O(n^2): every prefix summed from scratch with Python ints, then wrapped."""
    for kind, dt in ((inputs_mod.I32_FULL, "i32"), (inputs_mod.I8_FULL, "i8")):
        x = inputs_mod.fill_host(kind, 11, 0, n)
        xs = [int(v) for v in x]
        want_inc = [wrap32(sum(xs[:k + 1])) for k in range(n)]
        want_exc = [wrap32(sum(xs[:k])) for k in range(n)]
        assert oracle.inclusive(x, dt).tolist() == want_inc
        assert oracle.exclusive(x, dt).tolist() == want_exc


def test_bruteforce_float_exact(oracle):
    """Small-integer floats: every prefix is exact, so fsum of each prefix must
    equal the oracle's fp64 value bit for bit."""
    rng = np.random.default_rng(5)
    x = rng.integers(-1000, 1000, 1500).astype(np.float32)
    y64, a64, y32 = oracle.inclusive(x, "f32")
    for k in range(0, 1500, 7):
        assert y64[k] == math.fsum(float(v) for v in x[:k + 1])
        assert a64[k] == math.fsum(abs(float(v)) for v in x[:k + 1])


def test_int8_exhaustive_12bit_flags(oracle):
    """All 4096 length-12 0/1 flag patterns: inclusive_i = popcount(bits <= i)."""
    pats = np.arange(4096)
    X = ((pats[:, None] >> np.arange(12)[None, :]) & 1).astype(np.int8)
    for p in range(4096):
        y = oracle.inclusive(X[p], "i8")
        e = oracle.exclusive(X[p], "i8")
        for i in range(12):
            mask_le = (1 << (i + 1)) - 1
            assert y[i] == bin(p & mask_le).count("1")
            assert e[i] == bin(p & (mask_le >> 1)).count("1")


def test_int8_all_pairs(oracle):
    """All 65,536 int8 vectors of length 2: [a, a+b] and [0, a]."""
    a = np.repeat(np.arange(-128, 128), 256)
    b = np.tile(np.arange(-128, 128), 256)
    X = np.stack([a, b], 1).astype(np.int8)
    inc = oracle.rows(X, "i8")
    exc = oracle.rows(X, "i8", exclusive=True)
    assert np.array_equal(inc[:, 0], a) and np.array_equal(inc[:, 1], a + b)
    assert np.array_equal(exc[:, 0], 0 * a) and np.array_equal(exc[:, 1], a)


# ------------------------------------------------------------ invariants

def test_exclusive_invariant_and_totals(oracle, inputs_mod):
    n = 300001
    for kind, dt in ((inputs_mod.I32_FULL, "i32"), (inputs_mod.I8_FULL, "i8"),
                     (inputs_mod.I32_U100, "i32"), (inputs_mod.I8_FLAG, "i8")):
        x = inputs_mod.fill_host(kind, 3, 0, n)
        inc = oracle.inclusive(x, dt)
        exc = oracle.exclusive(x, dt)
        assert exc[0] == 0
        assert np.array_equal((exc.astype(np.int64) + x) & M32, inc.astype(np.int64) & M32)
        assert np.array_equal(exc[1:], inc[:-1])       # P461: shifted right by one
        tot = oracle.total(x, dt)
        assert tot == int(np.sum(x, dtype=np.int64))
        assert wrap32(tot) == int(inc[-1])
    f = inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n)
    e = oracle.exclusive(f, "i8")
    assert int(e[-1]) + int(f[-1]) == int(np.count_nonzero(f))


def test_float_exclusive_shift(oracle, inputs_mod):
    x = inputs_mod.fill_host(inputs_mod.F32_NORMAL, 9, 0, 5000)
    i64, ia, i32 = oracle.inclusive(x, "f32")
    e64, ea, e32 = oracle.exclusive(x, "f32")
    assert e64[0] == 0.0 and np.array_equal(e64[1:], i64[:-1])
    assert np.array_equal(ea, ia)       # A_i = sum_{j<=i}|x_j| for both (reading R6)


def test_carry_in(oracle, inputs_mod):
    x = inputs_mod.fill_host(inputs_mod.I32_FULL, 4, 0, 10000)
    c = -123456789
    assert np.array_equal(oracle.inclusive(x, "i32", carry_in=c).astype(np.int64) & M32,
                          (oracle.inclusive(x, "i32").astype(np.int64) + c) & M32)
    e = oracle.exclusive(x, "i32", carry_in=c)
    assert e[0] == c
    f = inputs_mod.fill_host(inputs_mod.F32_PM1, 4, 0, 10000)
    y64, a64, _ = oracle.inclusive(f, "f32", carry_in=-1000.0)
    assert np.array_equal(y64, -1000.0 + np.cumsum(f.astype(np.int64)))
    assert np.array_equal(a64, 1000.0 + np.cumsum(np.abs(f.astype(np.int64))))   # R6


def test_streaming_equals_whole(oracle, inputs_mod):
    n = 200003
    rng = np.random.default_rng(1)
    cuts = np.sort(rng.choice(np.arange(1, n), 17, replace=False))
    bounds = [0, *cuts.tolist(), n]
    for kind, dt in ((inputs_mod.I32_FULL, "i32"), (inputs_mod.I8_FULL, "i8")):
        x = inputs_mod.fill_host(kind, 8, 0, n)
        for exc in (False, True):
            whole = oracle.IntScan(dt)(x, exc)
            st = oracle.IntScan(dt)
            parts = np.concatenate([st(x[a:b], exc) for a, b in zip(bounds, bounds[1:])])
            assert np.array_equal(whole, parts)
    for kind, dt in ((inputs_mod.F32_NORMAL, "f32"), (inputs_mod.F16_U01, "f16")):
        x = inputs_mod.fill_host(kind, 8, 0, n)
        for exc in (False, True):
            whole = oracle.FloatScan(dt)(x, exc)
            st = oracle.FloatScan(dt)
            parts = [st(x[a:b], exc) for a, b in zip(bounds, bounds[1:])]
            for k in range(3):
                assert np.array_equal(whole[k], np.concatenate([p[k] for p in parts]))


def test_sharded_concat(oracle, inputs_mod):
    """RSS across shards: carry_r = sum of lower shard totals; concat == whole."""
    n, G = 100000, 4
    x = inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n)
    whole = oracle.exclusive(x, "i8")
    per = -(-n // G)
    shards = [x[r * per:min(n, (r + 1) * per)] for r in range(G)]
    totals = [oracle.total(s, "i8") for s in shards]
    outs = [oracle.exclusive(s, "i8", carry_in=sum(totals[:r])) for r, s in enumerate(shards)]
    assert np.array_equal(np.concatenate(outs), whole)


def test_sign_of_zero(oracle):
    """P68: y_1 = x_1, so the inclusive scan of [-0.0] is -0.0."""
    y64, _, y32 = oracle.inclusive(np.array([-0.0, -0.0], np.float32), "f32")
    assert math.copysign(1, y64[0]) == -1 and math.copysign(1, y32[0]) == -1


# --------------------------------------------------------------- fp16/fp

def test_f16_decode_exhaustive(oracle):
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([oracle.f16_to_f64(b) for b in bits.tolist()])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.array_equal(np.signbit(got[~nan]), np.signbit(ref[~nan]))


def test_c2_exact_fixed_point(oracle, inputs_mod):
    """C2-type data (fp16 multiples of 2^-24 in [0,1]): the exact prefix sums
    are int64 fixed point k*2^-24; the fp64 oracle must equal them bit for bit
    and its fp32 output must be their correctly rounded value."""
    n = 1 << 22
    h = inputs_mod.fill_host(inputs_mod.F16_U01, 1, 0, n)
    k = np.round(h.view(np.float16).astype(np.float64) * 2.0 ** 24).astype(np.int64)
    exact = np.cumsum(k)
    y64, a64, y32 = oracle.inclusive(h, "f16")
    assert np.array_equal(y64, exact.astype(np.float64) * 2.0 ** -24)
    assert np.array_equal(a64, y64)                            # all x >= 0
    assert np.array_equal(y32, (exact.astype(np.float64) * 2.0 ** -24).astype(np.float32))


def test_f32_pm1_exact(oracle, inputs_mod):
    x = inputs_mod.fill_host(inputs_mod.F32_PM1, 7, 0, 1 << 20)
    y64, a64, y32 = oracle.inclusive(x, "f32")
    c = np.cumsum(x.astype(np.int64))
    assert np.array_equal(y64, c) and np.array_equal(y32, c.astype(np.float32))
    assert np.array_equal(a64, np.cumsum(np.abs(x.astype(np.int64))))


def test_f32_total_within_bound(oracle, inputs_mod):
    """Sequential fp64 total vs the exactly rounded math.fsum: |err| <= n eps sum|x|."""
    x = inputs_mod.fill_host(inputs_mod.F32_NORMAL, 4, 0, 200000)
    t = oracle.total(x, "f32")
    exact = math.fsum(x.astype(np.float64).tolist())
    bound = len(x) * 2.0 ** -53 * float(np.abs(x.astype(np.float64)).sum())
    assert abs(t - exact) <= bound
    y64, _, _ = oracle.inclusive(x, "f32")
    assert y64[-1] == t


def test_tolerance_checker():
    import oracle as O
    rng = np.random.default_rng(0)
    ref = rng.normal(size=1000) * 100
    A = np.abs(ref) + 50.0
    tol = 1e-6 * A + 1e-6
    sign = np.where(rng.random(1000) < 0.5, -1.0, 1.0)
    ok = (ref + 0.5 * tol * sign)
    bad, worst, at = O.check_f32(ok.astype(np.float32), ok, A)   # exact vs itself
    assert bad == 0
    # float32 rounding of ok adds < 2^-24 |ok|; here tolerance-relative
    ref2 = ok.astype(np.float32).astype(np.float64)
    pert = ref2 + 0.99 * (1e-6 * A + 1e-6)
    bad, worst, at = O.check_f32(ref2.astype(np.float32), pert, A)
    assert bad == 0 and 0.98 < worst <= 0.99 + 1e-9
    pert = ref2 + 1.01 * (1e-6 * A + 1e-6)
    bad, worst, at = O.check_f32(ref2.astype(np.float32), pert, A)
    assert bad == 1000 and worst > 1.0
    got = np.array([np.nan, np.inf, 1.0], np.float32)
    bad, _, _ = O.check_f32(got, np.array([np.nan, np.inf, np.nan]), np.ones(3))
    assert bad == 1


# ------------------------------------- the paper's matrix formulation (pins)

def _U(s):
    return np.triu(np.ones((s, s), np.int64))


def test_eqn_scan_identity(oracle, inputs_mod):
    """Eq. (eqn:scan), P165-169: scan(z) = A@U_s + L^-_s@A@1_s for z viewed as
    an s x s row-major matrix A (zero padded).  Evaluated with int64 matmuls
    in the paper's order C1 = A@1, C2 = A@U, C2 += L^-@C1 (P171-177)."""
    for s, ell in ((4, 16), (8, 61), (16, 256), (32, 1000)):
        z = inputs_mod.fill_host(inputs_mod.I32_U100, s, 0, ell)
        A = np.zeros(s * s, np.int64)
        A[:ell] = z
        A = A.reshape(s, s)
        ones = np.ones((s, s), np.int64)
        Lm = np.tril(np.ones((s, s), np.int64), -1)
        C1 = A @ ones
        C2 = A @ _U(s)
        C2 = C2 + Lm @ C1
        assert np.array_equal(C2.reshape(-1)[:ell], oracle.inclusive(z, "i32"))


def test_alg1_scanu(oracle, inputs_mod):
    """Alg. 1 (ScanU, P141-163): per l-tile one A@U_s, then the vector unit adds
    the running `partial` to every s-row and takes its last entry."""
    s = 8
    n = 5 * s * s + 13
    x = inputs_mod.fill_host(inputs_mod.I32_U100, 21, 0, n).astype(np.int64)
    y = np.zeros(n, np.int64)
    partial = 0
    for t0 in range(0, n, s * s):
        tile = np.zeros(s * s, np.int64)
        m = min(s * s, n - t0)
        tile[:m] = x[t0:t0 + m]
        C = tile.reshape(s, s) @ _U(s)
        for r in range(s):
            C[r] += partial
            partial = C[r, -1]
        y[t0:t0 + m] = C.reshape(-1)[:m]
    assert np.array_equal(y, oracle.inclusive(x.astype(np.int32), "i32"))


def test_alg3_mcscan(oracle, inputs_mod):
    """Alg. 3 (MCScan, P229-261): Phase I local s-scans (A@U_s) and block sums r
    recomputed from x; SyncAll; Phase II partial = sum of r[:i], propagated over
    each block's s-tiles.  Also the exclusive variant of App. B.2 (P461)."""
    s, B = 4, 5
    n = 7 * s * s * B // 2 + 3
    x = inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n).astype(np.int64)
    per = -(-n // B)
    blocks = [(b * per, min(n, (b + 1) * per)) for b in range(B)]
    y = np.zeros(n, np.int64)
    r = np.zeros(B, np.int64)
    for b, (lo, hi) in enumerate(blocks):           # Phase I
        for t0 in range(lo, hi, s):
            row = np.zeros(s, np.int64)
            row[:min(s, hi - t0)] = x[t0:min(hi, t0 + s)]
            y[t0:min(hi, t0 + s)] = (row @ _U(s))[:min(s, hi - t0)]
        r[b] = x[lo:hi].sum()
    for b, (lo, hi) in enumerate(blocks):           # Phase II
        partial = r[:b].sum()
        for t0 in range(lo, hi, s):
            seg = slice(t0, min(hi, t0 + s))
            y[seg] += partial
            partial = y[seg][-1]
    assert np.array_equal(y, oracle.inclusive(x.astype(np.int8), "i8"))
    exc = np.concatenate([[0], y[:-1]])             # App. B.2 shift
    assert np.array_equal(exc, oracle.exclusive(x.astype(np.int8), "i8"))


def test_rows_equal_per_row(oracle, inputs_mod):
    X = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 0, 5, 1000)
    y64, a64, y32 = oracle.rows(X, "f32")
    for r in range(5):
        r64, ra, r32 = oracle.inclusive(X[r], "f32")
        assert np.array_equal(y64[r], r64) and np.array_equal(y32[r], r32)
    # softmax rows: non-decreasing and ending at 1 within fp32 rounding of p
    assert np.all(np.diff(y64, axis=1) >= 0)
    assert np.all(np.abs(y64[:, -1] - 1.0) < 1e-5)
    Xi = np.arange(24, dtype=np.int32).reshape(4, 6)
    Yi = oracle.rows(Xi, "i32")
    for r in range(4):
        assert np.array_equal(Yi[r], oracle.inclusive(Xi[r], "i32"))


def test_total_f16_pins(oracle, inputs_mod):
    """oracle_total_f16 (the checker of the GPU's fp16 scan_total / shard sums).
    C2-type data: every value is k*2^-24, so the exact total is an int64 count
    of 2^-24 units (< 2^53: exact in fp64) -- the fp64 sequential sum must equal
    it bit for bit.  N(0,1) fp16 data: within n*2^-53*sum|x| of math.fsum over
    numpy's own binary16 decode.  Specials: inf / NaN propagate."""
    n = 1 << 20
    h = inputs_mod.fill_host(inputs_mod.F16_U01, 1, 0, n)
    k = np.round(h.view(np.float16).astype(np.float64) * 2.0 ** 24).astype(np.int64)
    assert oracle.total(h, "f16") == float(int(k.sum())) * 2.0 ** -24
    g = inputs_mod.fill_host(inputs_mod.F16_NORMAL, 9, 0, 300001)
    v = g.view(np.float16).astype(np.float64)
    exact = math.fsum(v.tolist())
    assert abs(oracle.total(g, "f16") - exact) <= len(v) * 2.0 ** -53 * float(np.abs(v).sum())
    assert oracle.total(g, "f16") != oracle.total(g[:-1], "f16") or v[-1] == 0.0  # last element counted
    sp = np.array([0x3C00, 0x7C00, 0x3C00], np.uint16)              # 1, +inf, 1
    assert oracle.total(sp, "f16") == math.inf
    sp = np.array([0x7C00, 0xFC00], np.uint16)                      # +inf + -inf
    assert math.isnan(oracle.total(sp, "f16"))
    assert oracle.total(np.array([0x8001, 0x0001], np.uint16), "f16") == 0.0   # -/+ smallest subnormal
    assert oracle.total(np.array([0x0001] * 3, np.uint16), "f16") == 3 * 2.0 ** -24


@pytest.mark.parametrize("dt", ["i32", "f32"])
def test_rows_exclusive_pins(oracle, inputs_mod, dt):
    """The exclusive branch of oracle_rows_* (P461 per row, P437): brute force
    with Python integers (exact, mod 2^32 for int32; small-integer floats are
    exact in fp64), e[r][0] = 0 as +0.0, and e[r] = (0, inclusive shifted)."""
    R, C = 7, 333
    rng = np.random.default_rng(11)
    if dt == "i32":
        X = rng.integers(-(1 << 31), 1 << 31, (R, C), dtype=np.int64).astype(np.int32)
        E = oracle.rows(X, "i32", exclusive=True)
        I = oracle.rows(X, "i32")
        for r in range(R):
            acc = 0
            for i in range(C):
                assert E[r, i] == wrap32(acc), (r, i)
                acc += int(X[r, i])
            assert np.array_equal(E[r], np.concatenate([[0], I[r, :-1]]))
    else:
        X = rng.integers(-1000, 1001, (R, C)).astype(np.float32)
        e64, ea, e32 = oracle.rows(X, "f32", exclusive=True)
        i64, ia, i32 = oracle.rows(X, "f32")
        for r in range(R):
            acc = 0
            for i in range(C):
                assert e64[r, i] == float(acc) and e32[r, i] == np.float32(acc), (r, i)
                acc += int(X[r, i])
            assert not np.signbit(e64[r, 0])
            assert np.array_equal(e64[r, 1:], i64[r, :-1])
            # tolerance weight: A_i = sum_{j<=i}|x_j| for exclusive too (R7)
            assert np.array_equal(ea[r], np.cumsum(np.abs(X[r].astype(np.int64))).astype(np.float64))
        P = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 0, 3, 4096)
        p64, _, _ = oracle.rows(P, "f32", exclusive=True)
        q64, _, _ = oracle.rows(P, "f32")
        assert np.all(p64[:, 0] == 0.0) and np.array_equal(p64[:, 1:], q64[:, :-1])


@pytest.mark.parametrize("dt", ["i32", "i8", "f32", "f16"])
def test_threaded_baseline(oracle, inputs_mod, dt):
    """The all-core CPU baseline (oracle_threaded.c): integers bit-identical to
    the sequential oracle for any thread count and ragged chunking; floats
    within the north_star tolerance of the sequential fp64 scan."""
    kind = {"i32": inputs_mod.I32_FULL, "i8": inputs_mod.I8_FULL, "f32": inputs_mod.F32_NORMAL,
            "f16": inputs_mod.F16_NORMAL}[dt]
    for n in (1, 5, 1000, 100003):
        x = inputs_mod.fill_host(kind, n, 0, n)
        for T in (1, 2, 3, 8, 13):
            for exc in (False, True):
                got = oracle.scan_threaded(x, dt, exclusive=exc, threads=T)
                ref = (oracle.exclusive if exc else oracle.inclusive)(x, dt)
                if dt in ("i32", "i8"):
                    assert np.array_equal(got, ref), (n, T, exc)
                else:
                    bad, worst, _ = oracle.check_f32(got, ref[0], ref[1])
                    assert bad == 0, (n, T, exc, worst)
                    if T == 1:
                        assert np.array_equal(got, ref[2])


@pytest.mark.parametrize("dt", ["i32", "f32"])
def test_threaded_rows_baseline(oracle, inputs_mod, dt):
    """Row batches on T threads give exactly the sequential row oracle."""
    kind = inputs_mod.I32_FULL if dt == "i32" else inputs_mod.F32_NORMAL
    X = inputs_mod.fill_host(kind, 3, 0, 37 * 501).reshape(37, 501)
    ref = oracle.rows(X, dt)
    for T in (1, 4, 37, 64):
        got = oracle.scan_threaded_rows(X, dt, threads=T)
        assert np.array_equal(got, ref if dt == "i32" else ref[2]), T
