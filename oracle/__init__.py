"""Plain sequential CPU oracle for the prefix sum -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product package ``paper_2505_15112_b200`` never imports it, and it shares no
code with the CUDA kernels.

The arithmetic lives in ``oracle_scan.c`` (plain C, fp64 for floats, uint32
wrap for integers); this module only marshals numpy arrays through ctypes.
Every function cites the PAPER.md passage it follows (see oracle_scan.c's
header for the full list):

* P68  (Sec. 2)      inclusive prefix sum y_i = y_{i-1} + x_i, y_1 = x_1
* P461 (App. B.2)    exclusive = inclusive shifted right by one, 0 first
* P98, P459          fp16 -> fp32 and int8 -> int32 type pairs
* P437 (App. B.1)    batched scan = every row independently
* P73  (Sec. 2.1)    block reduction (the "R" of Reduce-Scan-Scan)

Parity pins: tests/test_oracle.py (closed forms, invariants, brute force,
exhaustive fp16 decode, exact fixed-point sums, SPEC/paper fixtures under
tests/golden/).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

I32, F32, F16, I8 = "i32", "f32", "f16", "i8"


class _IState(ctypes.Structure):
    _fields_ = [("sum", ctypes.c_uint32), ("count", ctypes.c_int64)]


class _FState(ctypes.Structure):
    _fields_ = [("sum", ctypes.c_double), ("abs_sum", ctypes.c_double),
                ("count", ctypes.c_int64), ("has_carry", ctypes.c_int)]


def build() -> str:
    """Compile liboracle.so with gcc (no fast-math, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("oracle_scan.c", "oracle_ops.c", "oracle_threaded.c")]
        if (not os.path.exists(_LIB_PATH)
                or os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(f) for f in srcs)):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.oracle_istate_init.argtypes = [ctypes.POINTER(_IState), I64]
        L.oracle_fstate_init.argtypes = [ctypes.POINTER(_FState), ctypes.c_double, I]
        for f in ("oracle_scan_i32", "oracle_scan_i8"):
            getattr(L, f).argtypes = [P, I64, I, ctypes.POINTER(_IState), P]
        for f in ("oracle_scan_f32", "oracle_scan_f16"):
            getattr(L, f).argtypes = [P, I64, I, ctypes.POINTER(_FState), P, P, P]
        L.oracle_f16_to_f64.argtypes = [ctypes.c_uint16]
        L.oracle_f16_to_f64.restype = ctypes.c_double
        for f in ("oracle_total_i32", "oracle_total_i8"):
            getattr(L, f).argtypes = [P, I64]
            getattr(L, f).restype = I64
        for f in ("oracle_total_f32", "oracle_total_f16"):
            getattr(L, f).argtypes = [P, I64]
            getattr(L, f).restype = ctypes.c_double
        L.oracle_check_f32.argtypes = [P, P, P, I64, ctypes.c_double, ctypes.c_double,
                                       ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_int64)]
        L.oracle_check_f32.restype = I64
        L.oracle_rows_f32.argtypes = [P, I64, I64, I64, I64, I, P, P, P]
        L.oracle_rows_i32.argtypes = [P, I64, I64, I64, I64, I, P]
        # oracle_threaded.c: the all-core CPU baseline (bench.py cpu_baseline only)
        L.oracle_scan_threaded.argtypes = [P, I64, I, I, I, P]
        L.oracle_scan_threaded.restype = I
        L.oracle_rows_threaded.argtypes = [P, I64, I64, I, I, I, P]
        L.oracle_rows_threaded.restype = I
        # oracle_ops.c: scan applications (Sec. 5, App. B.3)
        L.oracle_split.argtypes = [P, P, I64, I, I, P, P]
        L.oracle_split.restype = I64
        L.oracle_sort_encode.argtypes = [ctypes.c_uint32, I]
        L.oracle_sort_encode.restype = ctypes.c_uint32
        L.oracle_radix_sort.argtypes = [P, I64, I, I, P, P]
        L.oracle_weighted_sample.argtypes = [P, I64, ctypes.c_double]
        L.oracle_weighted_sample.restype = I64
        L.oracle_top_p_sample.argtypes = [P, I64, ctypes.c_double, ctypes.c_double,
                                          ctypes.POINTER(ctypes.c_int64)]
        L.oracle_top_p_sample.restype = I64
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


_IN_DTYPE = {I32: np.int32, I8: np.int8, F32: np.float32, F16: np.uint16}


def _as_input(x, dt):
    x = np.ascontiguousarray(x)
    if dt == F16 and x.dtype == np.float16:
        x = x.view(np.uint16)
    want = _IN_DTYPE[dt]
    if x.dtype != want:
        raise TypeError(f"oracle {dt} scan expects {np.dtype(want)}, got {x.dtype}")
    return x


class IntScan:
    """Streaming integer scan state (R1: sum mod 2^32).  int32 or int8 input."""

    def __init__(self, dt: str, carry_in: int = 0):
        assert dt in (I32, I8)
        self.dt = dt
        self.st = _IState()
        lib().oracle_istate_init(ctypes.byref(self.st), int(carry_in))

    def __call__(self, x, exclusive: bool = False) -> np.ndarray:
        x = _as_input(x, self.dt)
        y = np.empty(x.shape[0], dtype=np.int32)
        fn = lib().oracle_scan_i32 if self.dt == I32 else lib().oracle_scan_i8
        fn(_ptr(x), x.shape[0], int(exclusive), ctypes.byref(self.st), _ptr(y))
        return y


class FloatScan:
    """Streaming float scan state (R4: fp64 running sum, one RNE rounding)."""

    def __init__(self, dt: str, carry_in: float | None = None):
        assert dt in (F32, F16)
        self.dt = dt
        self.st = _FState()
        lib().oracle_fstate_init(ctypes.byref(self.st),
                                 0.0 if carry_in is None else float(carry_in),
                                 0 if carry_in is None else 1)

    def __call__(self, x, exclusive: bool = False, want64=True, want_abs=True,
                 want32=True):
        x = _as_input(x, self.dt)
        n = x.shape[0]
        y64 = np.empty(n, np.float64) if want64 else None
        a64 = np.empty(n, np.float64) if want_abs else None
        y32 = np.empty(n, np.float32) if want32 else None
        fn = lib().oracle_scan_f32 if self.dt == F32 else lib().oracle_scan_f16
        fn(_ptr(x), n, int(exclusive), ctypes.byref(self.st), _ptr(y64), _ptr(a64),
           _ptr(y32))
        return y64, a64, y32


def inclusive(x, dt: str, carry_in=None):
    """P68 inclusive scan of a whole array.  Ints -> int32; floats -> (y64, A, y32)."""
    if dt in (I32, I8):
        return IntScan(dt, 0 if carry_in is None else carry_in)(x, False)
    return FloatScan(dt, carry_in)(x, False)


def exclusive(x, dt: str, carry_in=None):
    """P461 exclusive scan of a whole array (0, or the carry-in, first)."""
    if dt in (I32, I8):
        return IntScan(dt, 0 if carry_in is None else carry_in)(x, True)
    return FloatScan(dt, 0.0 if carry_in is None else carry_in)(x, True)


_DT_CODE = {I32: 0, F32: 1, F16: 2, I8: 3}


def scan_threaded(x, dt: str, exclusive: bool = False, threads: int = 1, out=None):
    """All-core BASELINE (oracle_threaded.c): the scan split over
    `threads` host threads (chunk sums, ordered carries, chunk scans).  int32
    output for integer types (bit-identical to inclusive()/exclusive()), fp32
    for float types (fp64 carries; a timing baseline, never a checker)."""
    x = _as_input(x, dt)
    n = x.shape[0]
    if out is None:
        out = np.empty(n, np.int32 if dt in (I32, I8) else np.float32)
    rc = lib().oracle_scan_threaded(_ptr(x), n, _DT_CODE[dt], int(exclusive), int(threads), _ptr(out))
    if rc != 0:
        raise RuntimeError("oracle_scan_threaded failed")
    return out


def scan_threaded_rows(X, dt: str, exclusive: bool = False, threads: int = 1, out=None):
    """All-core BASELINE for row batches: rows split over `threads` host
    threads, each row scanned by the sequential oracle (identical results)."""
    X = np.ascontiguousarray(X)
    R, C = X.shape
    x = _as_input(X.reshape(-1), dt)
    if out is None:
        out = np.empty((R, C), np.int32 if dt in (I32, I8) else np.float32)
    rc = lib().oracle_rows_threaded(_ptr(x), R, C, _DT_CODE[dt], int(exclusive), int(threads), _ptr(out))
    if rc != 0:
        raise RuntimeError("oracle_rows_threaded failed")
    return out


def total(x, dt: str):
    """P73 RSS reduction: int64 (int types) or fp64 (float types) sum."""
    x = _as_input(x, dt)
    fn = {I32: lib().oracle_total_i32, I8: lib().oracle_total_i8,
          F32: lib().oracle_total_f32, F16: lib().oracle_total_f16}[dt]
    return fn(_ptr(x), x.shape[0])


def rows(X, dt: str, exclusive: bool = False):
    """P437 batched scan: every row of a 2-D array scanned independently."""
    X = np.ascontiguousarray(X)
    R, C = X.shape
    if dt == I32:
        X = _as_input(X.reshape(-1), I32).reshape(R, C)
        Y = np.empty((R, C), np.int32)
        lib().oracle_rows_i32(_ptr(X), R, C, C, C, int(exclusive), _ptr(Y))
        return Y
    if dt == F32:
        X = _as_input(X.reshape(-1), F32).reshape(R, C)
        y64 = np.empty((R, C), np.float64)
        a64 = np.empty((R, C), np.float64)
        y32 = np.empty((R, C), np.float32)
        lib().oracle_rows_f32(_ptr(X), R, C, C, C, int(exclusive), _ptr(y64), _ptr(a64),
                              _ptr(y32))
        return y64, a64, y32
    out = [(exclusive_fn if exclusive else inclusive)(X[r], dt) for r in range(R)]
    if dt in (I32, I8):
        return np.stack(out)
    return tuple(np.stack([o[k] for o in out]) for k in range(3))


exclusive_fn = exclusive


def f16_to_f64(bits: int) -> float:
    """R5: IEEE binary16 decode from the bit layout."""
    return lib().oracle_f16_to_f64(int(bits) & 0xFFFF)


def check_f32(got, ref64, abs_w, rel=1e-6, abs_tol=1e-6):
    """north_star tolerance |got - ref| <= rel*A_i + abs_tol.

    Returns (violations, max err/tol, index of the max)."""
    got = np.ascontiguousarray(got, dtype=np.float32).reshape(-1)
    ref64 = np.ascontiguousarray(ref64, dtype=np.float64).reshape(-1)
    abs_w = np.ascontiguousarray(abs_w, dtype=np.float64).reshape(-1)
    assert got.shape == ref64.shape == abs_w.shape
    worst = ctypes.c_double()
    at = ctypes.c_int64()
    bad = lib().oracle_check_f32(_ptr(got), _ptr(ref64), _ptr(abs_w), got.shape[0], rel,
                                 abs_tol, ctypes.byref(worst), ctypes.byref(at))
    return int(bad), float(worst.value), int(at.value)


# ---------------------------------------------------------------------------
# Scan applications (oracle_ops.c): PAPER.md Sec. 5.1-5.5 and App. B.3.
# ---------------------------------------------------------------------------
KEY_TYPES = {"u16": 0, "i16": 1, "f16": 2, "u32": 3, "i32": 4, "f32": 5}
_KEY_NP = {"u16": np.uint16, "i16": np.int16, "f16": np.float16, "u32": np.uint32,
           "i32": np.int32, "f32": np.float32}


def split(x, flags, compress: bool = False, with_idx: bool = True):
    """P281-285 SplitInd / Compress: stable split, flag-true items first (R12).

    Returns (z, idx, T): z has n items (split) or T items (compress)."""
    x = np.ascontiguousarray(x)
    f = np.ascontiguousarray(flags).view(np.int8) if np.asarray(flags).dtype != np.int8 \
        else np.ascontiguousarray(flags)
    n = x.shape[0]
    assert f.shape[0] == n
    z = np.empty_like(x)
    idx = np.empty(n, np.int32) if with_idx else None
    T = lib().oracle_split(_ptr(x), _ptr(f), n, x.dtype.itemsize, int(compress), _ptr(z),
                           _ptr(idx))
    if compress:
        return z[:T], (idx[:T] if with_idx else None), int(T)
    return z, idx, int(T)


def sort_encode(bits: int, key_type: str) -> int:
    """P287 float pre-processing (R13 for integers): order-preserving unsigned code."""
    return int(lib().oracle_sort_encode(int(bits) & 0xFFFFFFFF, KEY_TYPES[key_type]))


def radix_sort(keys, key_type: str, descending: bool = False):
    """P286-287 LSB radix sort by one split per bit (R13).  Returns (sorted keys, idx)."""
    k = np.ascontiguousarray(keys, dtype=_KEY_NP[key_type])
    out = np.empty_like(k)
    idx = np.empty(k.shape[0], np.int32)
    lib().oracle_radix_sort(_ptr(k), k.shape[0], KEY_TYPES[key_type], int(descending), _ptr(out),
                            _ptr(idx))
    return out, idx


def weighted_sample(w, theta: float) -> int:
    """P463 inverse transform sampling on the scan of w (R14)."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    return int(lib().oracle_weighted_sample(_ptr(w), w.shape[0], float(theta)))


def top_p_sample(probs, p: float, u: float):
    """P298-299 top-p (nucleus) sampling: sort, scan, nucleus, sample (R15).

    Returns (token index, nucleus size)."""
    q = np.ascontiguousarray(probs, dtype=np.float32)
    kept = ctypes.c_int64()
    tok = lib().oracle_top_p_sample(_ptr(q), q.shape[0], float(p), float(u), ctypes.byref(kept))
    return int(tok), int(kept.value)
