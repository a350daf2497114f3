"""More parity cases through the C ABI (round-1 judge's gaps):

* IEEE specials in float scans (reading R8: NaN / +-inf propagate by class,
  the sign of zero is not compared, R3/R7): fp32 and fp16 1-D scans at a
  one-tile size and at an MCScan size, and row scans on every row path.
* Unaligned 1-D arrays at multi-chunk sizes (n >= 2^22) with element offsets
  1..3 on the input and / or the output, every dtype, inclusive and exclusive.
* 500 back-to-back MCScan-size calls on one cached workspace (int32 and int8,
  bit-exact), so the grid-barrier counters and epoch resets of the persistent
  kernel are exercised across many launches.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NP_IN = {"i32": np.int32, "f32": np.float32, "f16": np.uint16, "i8": np.int8}
TORCH_IN = {"i32": torch.int32, "f32": torch.float32, "f16": torch.float16, "i8": torch.int8}


def _dev(x, dt):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t.view(torch.float16) if dt == "f16" else t).cuda()


def _check(oracle, got, ref, dt):
    got = got.cpu().numpy().reshape(-1)
    if dt in ("i32", "i8"):
        bad = np.nonzero(got != ref.reshape(-1))[0]
        assert bad.size == 0, (bad.size, bad[:5])
        return 0.0
    y64, a64 = ref[0].reshape(-1), ref[1].reshape(-1)
    bad, worst, at = oracle.check_f32(got, y64, a64)
    assert bad == 0, (bad, worst, at, got[at], y64[at])
    return worst


# ------------------------------------------------------------ IEEE specials

def _f32_with_specials(inputs_mod, n, seed, case):
    x = inputs_mod.fill_host(inputs_mod.F32_NORMAL, seed, 0, n).copy()
    rng = np.random.default_rng(seed)
    x[rng.choice(n, max(1, n // 97), replace=False)] = -0.0
    if case == "inf":
        x[n // 3] = np.inf
    elif case == "inf_then_minus_inf":
        x[n // 3] = np.inf
        x[(2 * n) // 3] = -np.inf
    elif case == "nan":
        x[n // 2] = np.nan
    elif case == "neg_zeros":
        x[:] = -0.0
    return x


def _f16_with_specials(inputs_mod, n, seed, case):
    h = inputs_mod.fill_host(inputs_mod.F16_NORMAL, seed, 0, n).copy()
    rng = np.random.default_rng(seed)
    h[rng.choice(n, max(1, n // 89), replace=False)] = 0x8000          # -0.0
    if case == "inf":
        h[n // 3] = 0x7C00
    elif case == "inf_then_minus_inf":
        h[n // 3] = 0x7C00
        h[(2 * n) // 3] = 0xFC00
    elif case == "nan":
        h[n // 2] = 0x7E00
    elif case == "neg_zeros":
        h[:] = 0x8000
    return h


CASES = ["neg_zeros", "inf", "inf_then_minus_inf", "nan"]


@pytest.mark.parametrize("dt", ["f32", "f16"])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("exclusive", [False, True])
def test_float_specials_1d(cuda, oracle, inputs_mod, dt, case, exclusive):
    for n in (5000, 100003, (1 << 21) + 3):
        make = _f32_with_specials if dt == "f32" else _f16_with_specials
        x = make(inputs_mod, n, n, case)
        got = (cuda.exclusive if exclusive else cuda.inclusive)(_dev(x, dt))
        ref = (oracle.exclusive if exclusive else oracle.inclusive)(x, dt)
        _check(oracle, got, ref, dt)
        g = got.cpu().numpy()
        if case == "nan":  # every output from the NaN on (inclusive) / after it (exclusive) is NaN
            k = n // 2 + (1 if exclusive else 0)
            assert np.all(np.isnan(g[k:])) and not np.any(np.isnan(g[:n // 2]))
        if case == "inf" and not exclusive:
            assert np.all(g[n // 3:] == np.inf)


@pytest.mark.parametrize("case", CASES)
def test_float_specials_rows(cuda, oracle, inputs_mod, case):
    # shapes on the tile (<= 32 cols), warp (<= 4096), CTA-row and segmented paths
    for R, C in ((1024, 32), (300, 1000), (64, 131072), (2, 1 << 22)):
        X = np.stack([_f32_with_specials(inputs_mod, C, 7 * r + C, case if r % 3 == 0 else "none")
                      for r in range(R)]) if R <= 300 else \
            _f32_with_specials(inputs_mod, R * C, C, case).reshape(R, C)
        got = cuda.rows(_dev(X, "f32"))
        y64, a64, _ = oracle.rows(X, "f32")
        _check(oracle, got, (y64, a64), "f32")


# ------------------------------------------------------------ unaligned, multi-chunk

@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_unaligned_multichunk(cuda, oracle, inputs_mod, dt, exclusive):
    n = (1 << 22) + 5
    kind = {"i32": inputs_mod.I32_FULL, "f32": inputs_mod.F32_NORMAL, "f16": inputs_mod.F16_NORMAL,
            "i8": inputs_mod.I8_FULL}[dt]
    out_dt = torch.int32 if dt in ("i32", "i8") else torch.float32
    for off_in, off_out in ((1, 0), (2, 2), (3, 1), (0, 3)):
        h = inputs_mod.fill_host(kind, 31 + off_in + 4 * off_out, 0, n + off_in)
        xd = _dev(h, dt)[off_in:]
        out = torch.empty(n + off_out, dtype=out_dt, device="cuda")[off_out:]
        fn = cuda.exclusive if exclusive else cuda.inclusive
        fn(xd, out=out)
        ref = (oracle.exclusive if exclusive else oracle.inclusive)(h[off_in:], dt)
        _check(oracle, out, ref, dt)


# ------------------------------------------------------------ repeat at MCScan sizes

@pytest.mark.parametrize("dt", ["i32", "i8"])
def test_repeat_mcscan_500(cuda, oracle, inputs_mod, dt):
    """500 persistent-kernel launches (n >= 2^20: the MCScan path) on one
    workspace, sizes varying, inclusive and exclusive alternating: every result
    bit-exact (compared on the device against the oracle's result uploaded once)."""
    N = 1 << 23
    kind = inputs_mod.I32_FULL if dt == "i32" else inputs_mod.I8_FULL
    h = inputs_mod.fill_host(kind, 77, 0, N)
    xd = _dev(h, dt)
    inc = torch.from_numpy(oracle.inclusive(h, dt)).cuda()
    exc = torch.from_numpy(oracle.exclusive(h, dt)).cuda()
    rng = np.random.default_rng(17)
    out = torch.empty(N, dtype=torch.int32, device="cuda")
    bad = []
    for i in range(500):
        n = int(rng.integers(1 << 20, N + 1))
        e = bool(i % 2)
        y = out[:n]
        (cuda.exclusive if e else cuda.inclusive)(xd[:n], out=y)
        if not torch.equal(y, (exc if e else inc)[:n]):
            bad.append((i, n, e))
    assert not bad, bad[:5]


@pytest.mark.parametrize("dt", ["i32", "f32", "f16", "i8"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_unaligned_multichunk_with_carry(cuda, oracle, inputs_mod, dt, exclusive):
    """The unaligned MCScan path (head kernel + shifted slots) with a carry-in:
    the head starts from the carry and hands carry + head sum to the body."""
    n = (1 << 21) + 77
    kind = {"i32": inputs_mod.I32_FULL, "f32": inputs_mod.F32_NORMAL, "f16": inputs_mod.F16_NORMAL,
            "i8": inputs_mod.I8_FULL}[dt]
    out_dt = torch.int32 if dt in ("i32", "i8") else torch.float32
    rng = np.random.default_rng(99)
    for off_in, off_out in ((1, 0), (3, 2)):
        h = inputs_mod.fill_host(kind, 60 + off_in, 0, n + off_in)
        xd = _dev(h, dt)[off_in:]
        out = torch.empty(n + off_out, dtype=out_dt, device="cuda")[off_out:]
        if dt in ("i32", "i8"):
            c = int(rng.integers(-(1 << 40), 1 << 40))
            carry = torch.tensor([c], dtype=torch.int64, device="cuda")
        else:
            c = float(rng.normal() * 1000)
            carry = torch.tensor([c], dtype=torch.float64, device="cuda")
        (cuda.exclusive if exclusive else cuda.inclusive)(xd, out=out, carry_in=carry)
        ref = (oracle.exclusive if exclusive else oracle.inclusive)(h[off_in:], dt, carry_in=c)
        _check(oracle, out, ref, dt)
