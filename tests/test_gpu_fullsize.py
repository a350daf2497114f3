"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (inputs generated on the device by the same recipe, the default
library path), against the streaming CPU oracle:

  C1 int32 inclusive + exclusive, n = 65,536, seed 0          -- every element
  C2 fp16 -> fp32 inclusive, n = 2^28, seed 1                 -- every element
  C3 int8 flags -> int32 exclusive, n = 2^30, seed 2          -- every element
  C4 rows 4096 x 131072 softmax(4 z), seed 3                  -- every element (64-row blocks)
  C5 fp32 inclusive, n = 2^32, seed 4                         -- every element: the oracle
                                                                 streams over all 2^32 elements
                                                                 in chunks of 2^26 (its running
                                                                 state is exact)
Integers bit-exact; floats |gpu - oracle_fp64| <= 1e-6 * A_i + 1e-6."""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 26


def _device_input(inputs_mod, kind, seed, n, dtype, cols=0, rows=0):
    if rows:
        x = torch.empty((rows, cols), dtype=dtype, device="cuda")
        inputs_mod.fill_device(kind, seed, 0, rows, cols, x)
    else:
        x = torch.empty(n, dtype=dtype, device="cuda")
        inputs_mod.fill_device(kind, seed, 0, n, 0, x)
    return x


def test_c1_full(cuda, oracle, inputs_mod):
    n = 65536
    x = _device_input(inputs_mod, inputs_mod.I32_U100, 0, n, torch.int32)
    xh = inputs_mod.fill_host(inputs_mod.I32_U100, 0, 0, n)
    assert np.array_equal(x.cpu().numpy(), xh)  # device and host generators agree
    assert np.array_equal(cuda.inclusive(x).cpu().numpy(), oracle.inclusive(xh, "i32"))
    assert np.array_equal(cuda.exclusive(x).cpu().numpy(), oracle.exclusive(xh, "i32"))


def _stream_check(cuda, oracle, inputs_mod, kind, seed, n, dtype, dt, exclusive, every=1, offset=0):
    x = _device_input(inputs_mod, kind, seed, n + offset, dtype)[offset:]
    y = (cuda.exclusive if exclusive else cuda.inclusive)(x)
    torch.cuda.synchronize()
    del x
    st = oracle.IntScan(dt) if dt in ("i32", "i8") else oracle.FloatScan(dt)
    worst, checked = 0.0, 0
    for k, lo in enumerate(range(0, n, CHUNK)):
        cnt = min(CHUNK, n - lo)
        xh = inputs_mod.fill_host(kind, seed, lo + offset, cnt)
        last = lo + cnt >= n
        if k % every and not last:
            st(xh, exclusive) if dt in ("i32", "i8") else st(xh, exclusive, want64=False, want_abs=False,
                                                              want32=False)
            continue
        got = y[lo:lo + cnt].cpu().numpy()
        if dt in ("i32", "i8"):
            ref = st(xh, exclusive)
            bad = np.nonzero(got != ref)[0]
            assert bad.size == 0, (lo, bad[:5])
        else:
            y64, a64, _ = st(xh, exclusive, want32=False)
            b, w, at = oracle.check_f32(got, y64, a64)
            assert b == 0, (lo, b, w, at)
            worst = max(worst, w)
        checked += 1
    return worst, checked


def test_c2_full(cuda, oracle, inputs_mod):
    worst, _ = _stream_check(cuda, oracle, inputs_mod, inputs_mod.F16_U01, 1, 1 << 28, torch.float16, "f16",
                             False)
    assert worst < 0.5


def test_c3_full(cuda, oracle, inputs_mod):
    _stream_check(cuda, oracle, inputs_mod, inputs_mod.I8_FLAG, 2, 1 << 30, torch.int8, "i8", True)


def test_c4_full(cuda, oracle, inputs_mod):
    R, C = 4096, 131072
    X = _device_input(inputs_mod, inputs_mod.F32_SOFTMAX, 3, 0, torch.float32, cols=C, rows=R)
    Y = cuda.rows(X)
    torch.cuda.synchronize()
    for r0 in range(0, R, 64):
        Xh = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, r0, 64, C)
        y64, a64, _ = oracle.rows(Xh, "f32")
        b, w, at = oracle.check_f32(Y[r0:r0 + 64].cpu().numpy(), y64, a64)
        assert b == 0, (r0, b, w, at)
        # softmax rows: every row sums to 1 within fp32 rounding, scans are non-decreasing
        assert np.all(np.abs(y64[:, -1] - 1.0) < 1e-5)


def test_c5_full(cuda, oracle, inputs_mod):
    worst, checked = _stream_check(cuda, oracle, inputs_mod, inputs_mod.F32_NORMAL, 4, 1 << 32, torch.float32,
                                   "f32", False)
    assert checked == (1 << 32) // CHUNK and worst < 0.5


def test_c3_unaligned_full(cuda, oracle, inputs_mod):
    """C3 on x[1:] (input one byte past a 16-byte boundary, fresh aligned output):
    the shifted-slot MCScan, every element bit-exact."""
    _stream_check(cuda, oracle, inputs_mod, inputs_mod.I8_FLAG, 2, (1 << 30) - 1, torch.int8, "i8", True, offset=1)


def test_c2_unaligned_full(cuda, oracle, inputs_mod):
    """C2 on x[3:] (fp16 input 6 bytes past a boundary): shifted-slot MCScan."""
    worst, _ = _stream_check(cuda, oracle, inputs_mod, inputs_mod.F16_U01, 1, (1 << 28) - 3, torch.float16, "f16",
                             False, offset=3)
    assert worst < 0.5
