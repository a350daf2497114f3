"""Seeded synthetic inputs for the scan workloads (no scan arithmetic here).

This is the one module both sides of a parity check use (DESIGN.md
"Inputs"): the oracle reads host arrays from ``fill_host``; the bench and the
GPU tests may fill device buffers with ``fill_device``.  Both evaluate the
same recipes from ``recipe.h`` with correctly rounded IEEE operations only,
so they are bit-identical (tests/test_inputs_gpu.py checks it on sampled
ranges).

The five BASELINE.json configs are described in ``CONFIGS``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

I32_U100, I8_FLAG, F16_U01, F32_NORMAL, F32_SOFTMAX = 0, 1, 2, 3, 4
I32_FULL, I8_FULL, F32_U01, F32_PM1, F16_NORMAL = 5, 6, 7, 8, 9

# numpy dtype of each recipe's elements (fp16 travels as raw uint16 bits)
KIND_DTYPE = {
    I32_U100: np.int32, I8_FLAG: np.int8, F16_U01: np.uint16, F32_NORMAL: np.float32,
    F32_SOFTMAX: np.float32, I32_FULL: np.int32, I8_FULL: np.int8, F32_U01: np.float32,
    F32_PM1: np.float32, F16_NORMAL: np.uint16,
}

# BASELINE.json configs[0..4]; dt = the scan type pair.
CONFIGS = {
    "C1": dict(name="C1_i32_n65536", kind=I32_U100, dt="i32", n=65536, rows=1, seed=0,
               ops=("inclusive", "exclusive"), multi_gpu=False),
    "C2": dict(name="C2_f16f32_n2^28", kind=F16_U01, dt="f16", n=1 << 28, rows=1, seed=1,
               ops=("inclusive",), multi_gpu=False),
    "C3": dict(name="C3_i8flag_i32_exc_n2^30", kind=I8_FLAG, dt="i8", n=1 << 30, rows=1,
               seed=2, ops=("exclusive",), multi_gpu=True),
    "C4": dict(name="C4_f32_rows4096x131072", kind=F32_SOFTMAX, dt="f32", n=131072,
               rows=4096, seed=3, ops=("inclusive",), multi_gpu=False),
    "C5": dict(name="C5_f32_n2^32", kind=F32_NORMAL, dt="f32", n=1 << 32, rows=1, seed=4,
               ops=("inclusive",), multi_gpu=True),
}

_host = None
_dev = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load(name):
    path = os.path.join(_HERE, name)
    srcs = [os.path.join(_HERE, f) for f in ("recipe.h", "softmax.h", "gen_host.c",
                                             "gen_device.cu")]
    if not os.path.exists(path) or os.path.getmtime(path) < max(map(os.path.getmtime, srcs)):
        build()
    return ctypes.CDLL(path)


def host_lib():
    global _host
    if _host is None:
        L = _load("libinputs_host.so")
        L.inputs_fill_host.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.inputs_fill_host.restype = ctypes.c_int
        _host = L
    return _host


def dev_lib():
    global _dev
    if _dev is None:
        L = _load("libinputs_dev.so")
        L.inputs_fill_device.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                         ctypes.c_void_p]
        L.inputs_fill_device.restype = ctypes.c_int
        _dev = L
    return _dev


def fill_host(kind: int, seed: int, start: int, n: int, cols: int = 0,
              threads: int | None = None) -> np.ndarray:
    """Elements [start, start+n) of recipe `kind` (rows for F32_SOFTMAX)."""
    L = host_lib()
    if kind == F32_SOFTMAX:
        out = np.empty((n, cols), np.float32)
        unit = cols
    else:
        out = np.empty(n, KIND_DTYPE[kind])
        unit = 1
    threads = threads or min(32, os.cpu_count() or 1)
    chunk = max(1, -(-n // threads))
    if kind != F32_SOFTMAX:
        chunk = max(chunk, 1 << 16)
    flat = out.reshape(-1)
    item = flat.itemsize

    def work(lo):
        cnt = min(chunk, n - lo)
        rc = L.inputs_fill_host(kind, seed, start + lo, cnt, cols,
                                ctypes.c_void_p(flat.ctypes.data + lo * unit * item))
        if rc != 0:
            raise ValueError(f"inputs_fill_host: bad kind {kind}")

    starts = list(range(0, n, chunk))
    if len(starts) <= 1:
        for lo in starts:
            work(lo)
    else:
        with ThreadPoolExecutor(len(starts)) as ex:
            list(ex.map(work, starts))
    return out


def fill_device(kind: int, seed: int, start: int, n: int, cols: int, tensor) -> None:
    """Fill a CUDA torch tensor (contiguous, right itemsize) on the current stream."""
    import torch
    assert tensor.is_cuda and tensor.is_contiguous()
    rc = dev_lib().inputs_fill_device(kind, seed, start, n, cols,
                                      ctypes.c_void_p(tensor.data_ptr()),
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"inputs_fill_device failed: {rc}")
