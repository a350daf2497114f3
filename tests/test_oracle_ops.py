"""Pins for the scan-application oracle (oracle/oracle_ops.c), CPU only.

Each operator is checked against something other than itself: numpy's stable
sort / boolean indexing / searchsorted (library routines the operator reduces
to), exhaustive small cases, closed-form special cases and invariants of the
definitions in PAPER.md Sec. 5 (P281-299) and App. B.3 (P463).
"""

import numpy as np
import pytest

import oracle


# ----------------------------------------------------------- split / compress
def _np_split(x, f):
    """Stable partition via numpy's stable argsort on the key (flag == 0)."""
    order = np.argsort((f == 0).astype(np.int8), kind="stable")
    return x[order], order.astype(np.int32), int(np.count_nonzero(f))


@pytest.mark.parametrize("dtype", [np.int8, np.uint16, np.float32, np.int64])
@pytest.mark.parametrize("n", [0, 1, 7, 1000, 65537])
def test_split_matches_stable_partition(dtype, n):
    rng = np.random.default_rng(n)
    x = rng.integers(-1000, 1000, n).astype(dtype)
    f = rng.integers(0, 2, n).astype(np.int8)
    z, idx, T = oracle.split(x, f)
    zr, ir, Tr = _np_split(x, f)
    assert T == Tr
    assert np.array_equal(z, zr) and np.array_equal(idx, ir)
    zc, ic, Tc = oracle.split(x, f, compress=True)
    assert Tc == T and np.array_equal(zc, x[f != 0]) and np.array_equal(ic, np.nonzero(f)[0])


def test_split_exhaustive_length12():
    """All 4096 flag patterns of length 12 (P281: true first, stable)."""
    x = np.arange(12, dtype=np.int32)
    for bits in range(1 << 12):
        f = np.array([(bits >> i) & 1 for i in range(12)], np.int8)
        z, idx, T = oracle.split(x, f)
        assert T == bin(bits).count("1")
        trues = [i for i in range(12) if f[i]]
        falses = [i for i in range(12) if not f[i]]
        assert list(z) == trues + falses and list(idx) == trues + falses


def test_split_nonzero_flags_are_true():
    """R12: any nonzero int8 flag is true (not summed)."""
    x = np.arange(6, dtype=np.uint16)
    f = np.array([0, -3, 2, 0, 127, 0], np.int8)
    z, idx, T = oracle.split(x, f)
    assert T == 3 and list(z) == [1, 2, 4, 0, 3, 5]


def test_split_degenerate():
    x = np.arange(100, dtype=np.float32)
    for f in (np.ones(100, np.int8), np.zeros(100, np.int8)):
        z, idx, T = oracle.split(x, f)
        assert np.array_equal(z, x) and np.array_equal(idx, np.arange(100))
        assert T == int(f.sum())


# ----------------------------------------------------------------- radix sort
@pytest.mark.parametrize("kt", ["u16", "i16", "u32", "i32"])
@pytest.mark.parametrize("desc", [False, True])
def test_radix_sort_integers_match_numpy_stable(kt, desc):
    rng = np.random.default_rng(7)
    dt = {"u16": np.uint16, "i16": np.int16, "u32": np.uint32, "i32": np.int32}[kt]
    info = np.iinfo(dt)
    k = rng.integers(info.min, info.max, 5000, endpoint=True, dtype=np.int64).astype(dt)
    k[::7] = k[3]  # many ties: stability matters
    out, idx = oracle.radix_sort(k, kt, descending=desc)
    key = k.astype(np.int64)
    order = np.argsort(-key if desc else key, kind="stable")
    assert np.array_equal(idx, order) and np.array_equal(out, k[order])


@pytest.mark.parametrize("kt", ["f16", "f32"])
def test_radix_sort_floats_match_numpy(kt):
    rng = np.random.default_rng(11)
    dt = np.float16 if kt == "f16" else np.float32
    k = (rng.standard_normal(4000) * 100).astype(dt)
    k[::5] = k[1]
    k[k == 0] = dt(1)  # no signed zeros here (R13 orders -0 < +0; numpy ties them)
    for desc in (False, True):
        out, idx = oracle.radix_sort(k, kt, descending=desc)
        order = np.argsort(-k.astype(np.float64) if desc else k, kind="stable")
        assert np.array_equal(idx, order)
        assert np.array_equal(out.view(np.uint16 if kt == "f16" else np.uint32),
                              k[order].view(np.uint16 if kt == "f16" else np.uint32))


def test_radix_sort_f16_exhaustive_total_order():
    """All 65,536 fp16 bit patterns: P287's encoding yields the IEEE total order
    (R13): -NaN < -inf < ... < -0 < +0 < ... < +inf < +NaN."""
    rng = np.random.default_rng(3)
    bits = rng.permutation(np.arange(1 << 16, dtype=np.uint32)).astype(np.uint16)
    out, idx = oracle.radix_sort(bits.view(np.float16), "f16")
    ob = out.view(np.uint16)
    assert np.array_equal(bits[idx], ob)
    v = ob.view(np.float16).astype(np.float64)
    neg = (ob >> 15) == 1
    nan = np.isnan(v)
    # negative NaNs first, positive NaNs last, numbers in between non-decreasing
    n_negnan = int(np.count_nonzero(nan & neg))
    n_posnan = int(np.count_nonzero(nan & ~neg))
    assert nan[:n_negnan].all() and nan[len(v) - n_posnan:].all()
    mid = v[n_negnan:len(v) - n_posnan]
    assert not np.isnan(mid).any() and np.all(np.diff(mid) >= 0)
    zeros = np.nonzero(mid == 0)[0]
    assert list(ob[n_negnan + zeros]) == [0x8000, 0x0000]  # -0 before +0


def test_sort_encode_closed_form():
    """P287: positive -> MSB inverted, negative -> all bits inverted."""
    assert oracle.sort_encode(0x3C00, "f16") == 0xBC00      # +1.0
    assert oracle.sort_encode(0xBC00, "f16") == 0x43FF      # -1.0
    assert oracle.sort_encode(0x8000, "f16") == 0x7FFF      # -0
    assert oracle.sort_encode(0x0000, "f16") == 0x8000      # +0
    assert oracle.sort_encode(0x3F800000, "f32") == 0xBF800000
    assert oracle.sort_encode(0xBF800000, "f32") == 0x407FFFFF
    assert oracle.sort_encode(0x80000000, "i32") == 0 and oracle.sort_encode(0x7FFFFFFF, "i32") == 0xFFFFFFFF


# --------------------------------------------------------- weighted sampling
def test_weighted_sample_matches_searchsorted():
    rng = np.random.default_rng(5)
    for n in (1, 2, 17, 5000):
        w = rng.random(n).astype(np.float32)
        w[rng.random(n) < 0.2] = 0  # zero weights are never drawn
        if w.sum() == 0:
            w[0] = 1
        S = np.cumsum(w.astype(np.float64))
        for theta in (0.0, 0.25, 0.5, 0.999999, rng.random()):
            got = oracle.weighted_sample(w, theta)
            assert got == int(np.searchsorted(S, theta * S[-1], side="right"))
            assert w[got] > 0


def test_weighted_sample_frequencies_brute_force():
    """Inverse transform: over a fine theta grid each index is drawn in
    proportion to its weight (P463)."""
    w = np.array([1, 0, 3, 2, 0, 4], np.float32)
    G = 10000
    counts = np.zeros(len(w))
    for k in range(G):
        counts[oracle.weighted_sample(w, (k + 0.5) / G)] += 1
    assert np.allclose(counts / G, w / w.sum(), atol=1e-3)


# ------------------------------------------------------------------- top-p
def test_top_p_special_cases():
    rng = np.random.default_rng(9)
    q = rng.random(1000).astype(np.float32)
    q /= q.sum()
    # p = 0: greedy -- the (first) most probable token
    for u in (0.0, 0.5, 0.99):
        tok, K = oracle.top_p_sample(q, 0.0, u)
        assert K == 1 and tok == int(np.argmax(q))
    # p > total mass: nothing is cut, = weighted sampling in descending order
    order = np.argsort(-q.astype(np.float64), kind="stable")
    for u in (0.0, 0.3, 0.7, 0.999):
        tok, K = oracle.top_p_sample(q, 2.0, u)
        assert K == 1000 and tok == order[oracle.weighted_sample(q[order], u)]


def test_top_p_nucleus_is_minimal_and_sampled_in_proportion():
    rng = np.random.default_rng(13)
    q = np.exp(4 * rng.standard_normal(300)).astype(np.float32)
    q /= q.sum()
    s = np.sort(q.astype(np.float64))[::-1]
    for p in (0.1, 0.5, 0.9, 0.95):
        _, K = oracle.top_p_sample(q, p, 0.5)
        # smallest prefix of the descending order whose mass reaches p (R15)
        assert s[:K - 1].sum() < p <= s[:K].sum() + 1e-12
        G = 4000
        hits = {}
        for k in range(G):
            t, _ = oracle.top_p_sample(q, p, (k + 0.5) / G)
            hits[t] = hits.get(t, 0) + 1
        top = np.argsort(-q.astype(np.float64), kind="stable")[:K]
        assert set(hits) <= set(top.tolist())
        mass = q[top].astype(np.float64).sum()
        for t in top:
            assert abs(hits.get(int(t), 0) / G - q[t] / mass) <= 1.5 / G + 1e-9
