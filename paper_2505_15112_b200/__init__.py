"""B200-native device-wide prefix sum (scan): thin Python binding of libscan.so.

The product is the C ABI in ``include/scan.h`` (built from ``csrc/`` for
sm_100a).  This module only marshals torch tensors (device memory) and the
current CUDA stream into those calls; every step of the scan runs in the CUDA
kernels.  There is no CPU fallback: if ``libscan.so`` is missing or the device
is not a B200, the calls raise.

Public API (names follow the C ABI):
    inclusive(x, out=None, carry_in=None)     -- P68 inclusive prefix sum
    exclusive(x, out=None, carry_in=None)     -- P461 exclusive prefix sum
    rows(X, exclusive=False, out=None)        -- P437 batched row scan
    total(x)                                  -- RSS reduction (P73)
    carry_from_totals(totals, rank)           -- sum of lower shard totals
    sharded_inclusive / sharded_exclusive     -- see paper_2505_15112_b200.dist
    split(x, flags) / compress(x, flags)      -- P281-285 SplitInd / compress
    radix_sort(keys, descending=False)        -- P286-287 LSB radix sort by splits
    weighted_sample(w, theta)                 -- P463 inverse transform on scan(w)
    top_p_sample(probs, p, u)                 -- P298-299 sort + row scan + nucleus draw
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCAN_LIB selects another in-tree build of the same library (the tests' stress
# tier loads libscan_fuzz.so); a bare file name inside this package only.
LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ.get("SCAN_LIB", "libscan.so")))

SCAN_I32_I32, SCAN_F32_F32, SCAN_F16_F32, SCAN_I8_I32 = 0, 1, 2, 3
_STATUS = {0: "SCAN_OK", 1: "SCAN_ERR_ARG", 2: "SCAN_ERR_WORKSPACE", 3: "SCAN_ERR_CUDA",
           4: "SCAN_ERR_DEVICE"}

# input torch dtype -> (scan dtype code, output torch dtype, total/carry dtype)
DTYPES = {
    torch.int32: (SCAN_I32_I32, torch.int32, torch.int64),
    torch.float32: (SCAN_F32_F32, torch.float32, torch.float64),
    torch.float16: (SCAN_F16_F32, torch.float32, torch.float64),
    torch.int8: (SCAN_I8_I32, torch.int32, torch.int64),
}

_lib = None
_lock = threading.Lock()


class ScanError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load the in-tree libscan.so (build it with ``make -C paper_2505_15112_b200``)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ScanError(f"{LIB_PATH} not built; run __graft_entry__.build() or "
                            f"make -C {_HERE}")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
        L.scan_abi_version.restype = I
        L.scan_status_string.argtypes = [I]
        L.scan_status_string.restype = ctypes.c_char_p
        L.scan_workspace_bytes.argtypes = [I, I64]
        L.scan_workspace_bytes.restype = SZ
        L.scan_rows_workspace_bytes.argtypes = [I, I64, I64]
        L.scan_rows_workspace_bytes.restype = SZ
        L.scan_workspace_init.argtypes = [P, SZ, P]
        L.scan_workspace_init.restype = I
        for f in (L.scan_inclusive, L.scan_exclusive):
            f.argtypes = [P, P, I64, I, P, P, SZ, P]
            f.restype = I
        L.scan_rows.argtypes = [P, P, I64, I64, I64, I64, I, I, P, SZ, P]
        L.scan_rows.restype = I
        L.scan_total.argtypes = [P, I64, I, P, P, SZ, P]
        L.scan_total.restype = I
        L.scan_carry_from_totals.argtypes = [P, I, I, I, P, P]
        L.scan_carry_from_totals.restype = I
        L.scan_launch_count.restype = ctypes.c_uint64
        L.scan_host_stage_bytes.argtypes = [I, I64]
        L.scan_host_stage_bytes.restype = SZ
        L.scan_host.argtypes = [P, P, I64, I, I, I64, P, SZ, P, SZ, P]
        L.scan_host.restype = I
        L.scan_widen_copy.argtypes = [P, P, I64, I, P]
        L.scan_widen_copy.restype = I
        L.scan_shard_workspace_bytes.argtypes = [I, I64]
        L.scan_shard_workspace_bytes.restype = SZ
        L.scan_shard_reduce.argtypes = [P, I64, I, P, P, SZ, P]
        L.scan_shard_reduce.restype = I
        L.scan_shard_scan.argtypes = [P, P, I64, I, I, P, P, SZ, P]
        L.scan_shard_scan.restype = I
        L.scan_peer_slots_bytes.argtypes = [I]
        L.scan_peer_slots_bytes.restype = SZ
        L.scan_shard_reduce_publish.argtypes = [P, I64, I, P, P, I, I, ctypes.c_uint32, P, SZ, P]
        L.scan_shard_reduce_publish.restype = I
        L.scan_shard_scan_peers.argtypes = [P, P, I64, I, I, P, I, I, ctypes.c_uint32, P, SZ, P]
        L.scan_shard_scan_peers.restype = I
        # include/scan_ops.h
        L.scan_split_workspace_bytes.argtypes = [I64]
        L.scan_split_workspace_bytes.restype = SZ
        L.scan_split.argtypes = [P, P, P, P, I64, I, I, P, P, SZ, P]
        L.scan_split.restype = I
        L.scan_radix_sort_workspace_bytes.argtypes = [I64, I]
        L.scan_radix_sort_workspace_bytes.restype = SZ
        L.scan_radix_sort.argtypes = [P, P, P, I64, I, I, P, SZ, P]
        L.scan_radix_sort.restype = I
        L.scan_radix_sort_rows_workspace_bytes.argtypes = [I64, I64, I]
        L.scan_radix_sort_rows_workspace_bytes.restype = SZ
        L.scan_radix_sort_rows.argtypes = [P, P, P, I64, I64, I, I, P, SZ, P]
        L.scan_radix_sort_rows.restype = I
        L.scan_weighted_sample.argtypes = [P, I64, ctypes.c_double, P, P, P, SZ, P]
        L.scan_weighted_sample.restype = I
        L.scan_top_p_draw.argtypes = [P, P, I64, I64, I64, I64, ctypes.c_float, P, P, P, P]
        L.scan_top_p_draw.restype = I
        L.scan_top_p_sample.argtypes = [P, I64, I64, I64, ctypes.c_float, P, P, P, P, SZ, P]
        L.scan_top_p_sample.restype = I
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = load().scan_status_string(rc).decode()
        raise ScanError(f"{what}: {msg}")


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Workspace:
    """A caller-owned, initialised workspace (device uint8 buffer).

    One per (device, stream, kind) is cached by ``workspace()``; it grows on
    demand and is re-initialised (scan_workspace_init) whenever it is
    reallocated.  The buffer is allocated on the stream that uses it, so the
    caching allocator never hands its memory to another stream while kernels
    queued there may still touch it."""

    def __init__(self, nbytes: int, device, stream=None):
        nbytes = max(int(nbytes), 1 << 17)  # >= the header block (kWsDescOffset)
        s = stream if stream is not None else torch.cuda.current_stream(device)
        with torch.cuda.stream(s):
            self.buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
        off = (-self.buf.data_ptr()) % 256
        self.nbytes = nbytes
        self.ptr = self.buf.data_ptr() + off
        _check(load().scan_workspace_init(ctypes.c_void_p(self.ptr), nbytes, _stream_ptr(stream)),
               "scan_workspace_init")


_ws_cache: dict = {}


def workspace(nbytes: int, device=None, stream=None, kind: str = "scan") -> Workspace:
    """The cached workspace of (device, stream, kind).  Scans and the scan
    operators (kind="ops": split / compress / sort / top-p) keep separate
    buffers, so operator scratch never sits where a scan's look-back
    descriptors go (the C library also clears such scratch, see scan.h)."""
    dev = torch.device(device) if device is not None else torch.device("cuda",
                                                                       torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev.index, s.cuda_stream, kind)
    ws = _ws_cache.get(key)
    if ws is None or ws.nbytes < nbytes:
        ws = Workspace(max(nbytes, 2 * (ws.nbytes if ws else 0)), dev, s)
        _ws_cache[key] = ws
    return ws


def _prep(x: torch.Tensor):
    if not x.is_cuda:
        raise ScanError("input must be a CUDA tensor (there is no CPU path)")
    if x.dtype not in DTYPES:
        raise ScanError(f"unsupported input dtype {x.dtype}; use int32, float32, float16, int8")
    return DTYPES[x.dtype]


def _scan1d(x: torch.Tensor, out, carry_in, exclusive: bool, stream=None):
    dt, odt, cdt = _prep(x)
    if x.dim() != 1:
        raise ScanError("1-D scan expects a 1-D tensor; use rows() for batches")
    if not x.is_contiguous():
        raise ScanError("input must be contiguous")
    n = x.numel()
    if out is None:
        out = torch.empty(n, dtype=odt, device=x.device)
    elif out.dtype != odt or out.numel() != n or not out.is_contiguous():
        raise ScanError(f"out must be a contiguous {odt} tensor of {n} elements")
    if carry_in is not None and (carry_in.dtype != cdt or not carry_in.is_cuda):
        raise ScanError(f"carry_in must be a CUDA {cdt} tensor")
    L = load()
    ws = workspace(L.scan_workspace_bytes(dt, n), x.device, stream)
    fn = L.scan_exclusive if exclusive else L.scan_inclusive
    _check(fn(_ptr(x), _ptr(out), n, dt, _ptr(carry_in), ctypes.c_void_p(ws.ptr), ws.nbytes,
              _stream_ptr(stream)), "scan_exclusive" if exclusive else "scan_inclusive")
    return out


def inclusive(x: torch.Tensor, out=None, carry_in=None, stream=None) -> torch.Tensor:
    """Inclusive prefix sum (P68) of a 1-D CUDA tensor; int32 or fp32 result."""
    return _scan1d(x, out, carry_in, False, stream)


def exclusive(x: torch.Tensor, out=None, carry_in=None, stream=None) -> torch.Tensor:
    """Exclusive prefix sum (P461): out[0] = carry (0), out[i] = sum of x[:i]."""
    return _scan1d(x, out, carry_in, True, stream)


def rows(X: torch.Tensor, exclusive: bool = False, out=None, stream=None) -> torch.Tensor:
    """Scan every row of a 2-D CUDA tensor independently (P437).  Rows may be
    strided (row stride >= cols, unit column stride)."""
    dt, odt, _ = _prep(X)
    if X.dim() != 2 or (X.shape[1] > 1 and X.stride(1) != 1):
        raise ScanError("rows() expects a 2-D tensor with unit column stride")
    R, C = X.shape
    if R > 1 and X.stride(0) < C:  # expanded / overlapping rows: scan a dense copy
        X = X.contiguous()
    if out is None:
        out = torch.empty((R, C), dtype=odt, device=X.device)
    elif out.dtype != odt or tuple(out.shape) != (R, C) or (C > 1 and out.stride(1) != 1):
        raise ScanError(f"out must be a {odt} tensor of shape {(R, C)} with unit column stride")
    elif R > 1 and out.stride(0) < C:
        raise ScanError("out rows overlap (row stride < cols)")
    in_stride = X.stride(0) if R > 1 else C
    out_stride = out.stride(0) if R > 1 else C
    L = load()
    ws = workspace(L.scan_rows_workspace_bytes(dt, R, C), X.device, stream)
    _check(L.scan_rows(_ptr(X), _ptr(out), R, C, in_stride, out_stride, dt,
                       int(bool(exclusive)), ctypes.c_void_p(ws.ptr), ws.nbytes,
                       _stream_ptr(stream)), "scan_rows")
    return out


def total(x: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """Sum of a 1-D CUDA tensor: int64 (integer inputs) or fp64 (float inputs)."""
    dt, _, cdt = _prep(x)
    if out is None:
        out = torch.empty(1, dtype=cdt, device=x.device)
    L = load()
    ws = workspace(L.scan_workspace_bytes(dt, 0), x.device, stream)
    _check(L.scan_total(_ptr(x), x.numel(), dt, _ptr(out), ctypes.c_void_p(ws.ptr), ws.nbytes,
                        _stream_ptr(stream)), "scan_total")
    return out


def carry_from_totals(totals: torch.Tensor, rank: int, in_dtype: torch.dtype, out=None,
                      stream=None) -> torch.Tensor:
    """totals[0] + ... + totals[rank-1] (device), ready to use as carry_in."""
    dt, _, cdt = DTYPES[in_dtype]
    if totals.dtype != cdt:
        raise ScanError(f"totals must be {cdt}")
    if out is None:
        out = torch.empty(1, dtype=cdt, device=totals.device)
    _check(load().scan_carry_from_totals(_ptr(totals), totals.numel(), rank, dt, _ptr(out),
                                         _stream_ptr(stream)), "scan_carry_from_totals")
    return out


_stage_cache: dict = {}


def host_scan(h_in: torch.Tensor, h_out=None, exclusive: bool = False, chunk: int = 1 << 26,
              device=None, stream=None) -> torch.Tensor:
    """End-to-end scan of a HOST tensor (pin it for full speed): streamed
    through the GPU in chunks with H2D copy, scan and D2H copy overlapped
    (C ABI scan_host).  Returns the host output tensor once complete."""
    if h_in.is_cuda:
        raise ScanError("host_scan expects a CPU tensor; use inclusive()/exclusive() for device data")
    dt, odt, _ = DTYPES[h_in.dtype] if h_in.dtype in DTYPES else (None, None, None)
    if dt is None:
        raise ScanError(f"unsupported input dtype {h_in.dtype}")
    h_in = h_in.reshape(-1)
    n = h_in.numel()
    if h_out is None:
        h_out = torch.empty(n, dtype=odt, pin_memory=h_in.is_pinned())
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    chunk = max(1, min(int(chunk), max(n, 1)))
    L = load()
    sb = L.scan_host_stage_bytes(dt, chunk)
    key = (dev.index, sb)
    stage = _stage_cache.get(key)
    if stage is None:
        stage = torch.empty(sb, dtype=torch.uint8, device=dev)
        _stage_cache.clear()
        _stage_cache[key] = stage
    ws = workspace(L.scan_workspace_bytes(dt, chunk), dev, stream)
    _check(L.scan_host(ctypes.c_void_p(h_in.data_ptr()), ctypes.c_void_p(h_out.data_ptr()), n, dt,
                       int(bool(exclusive)), chunk, _ptr(stage), sb, ctypes.c_void_p(ws.ptr), ws.nbytes,
                       _stream_ptr(stream)), "scan_host")
    return h_out


def shard_workspace(x: torch.Tensor, stream=None) -> Workspace:
    """A fresh initialised workspace for one shard of the two-pass sharded scan
    (it keeps the shard's block sums between shard_reduce and shard_scan)."""
    dt, _, _ = _prep(x)
    return Workspace(load().scan_shard_workspace_bytes(dt, x.numel()), x.device, stream)


def shard_reduce(x: torch.Tensor, ws: Workspace | None = None, out=None, stream=None) -> torch.Tensor:
    """Pass 1 of the sharded scan (P73 block-level reduction): the shard total
    (1-element int64 / float64 CUDA tensor); block sums stay in `ws`."""
    dt, _, cdt = _prep(x)
    n = x.reshape(-1).numel()
    L = load()
    ws = ws if ws is not None else workspace(L.scan_shard_workspace_bytes(dt, n), x.device, stream)
    out = torch.empty(1, dtype=cdt, device=x.device) if out is None else out
    _check(L.scan_shard_reduce(_ptr(x), n, dt, _ptr(out), ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)),
           "scan_shard_reduce")
    return out


def shard_scan(x: torch.Tensor, exclusive: bool = False, carry_in=None, ws: Workspace | None = None, out=None,
               stream=None) -> torch.Tensor:
    """Pass 2 of the sharded scan: scan of the shard given to shard_reduce (same
    `ws`), every block starting from carry_in + its block prefix."""
    dt, odt, cdt = _prep(x)
    x = x.reshape(-1)
    n = x.numel()
    if carry_in is not None and (carry_in.dtype != cdt or not carry_in.is_cuda):
        raise ScanError(f"carry_in must be a CUDA {cdt} tensor")
    out = torch.empty(n, dtype=odt, device=x.device) if out is None else out
    L = load()
    ws = ws if ws is not None else workspace(L.scan_shard_workspace_bytes(dt, n), x.device, stream)
    _check(L.scan_shard_scan(_ptr(x), _ptr(out), n, dt, int(bool(exclusive)), _ptr(carry_in),
                             ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)), "scan_shard_scan")
    return out


def peer_slots_bytes(G: int) -> int:
    """Bytes of one rank's slot array for the device-initiated totals exchange."""
    return int(load().scan_peer_slots_bytes(G))


def shard_reduce_publish(x: torch.Tensor, peers_dev_ptr: int, G: int, rank: int, epoch: int,
                         ws: Workspace | None = None, out=None, stream=None) -> torch.Tensor:
    """shard_reduce + the total written straight into every rank's slot array
    (`peers_dev_ptr`: device address of G device pointers, rank q's slots as
    mapped on this GPU)."""
    dt, _, cdt = _prep(x)
    n = x.reshape(-1).numel()
    L = load()
    ws = ws if ws is not None else workspace(L.scan_shard_workspace_bytes(dt, n), x.device, stream)
    out = torch.empty(1, dtype=cdt, device=x.device) if out is None else out
    _check(L.scan_shard_reduce_publish(_ptr(x), n, dt, _ptr(out), ctypes.c_void_p(peers_dev_ptr), G, rank, epoch,
                                       ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)),
           "scan_shard_reduce_publish")
    return out


def shard_scan_peers(x: torch.Tensor, exclusive: bool, slots: torch.Tensor, G: int, rank: int, epoch: int,
                     ws: Workspace | None = None, out=None, stream=None) -> torch.Tensor:
    """shard_scan whose carry is read (in-kernel) from this rank's slot array."""
    dt, odt, _ = _prep(x)
    x = x.reshape(-1)
    n = x.numel()
    out = torch.empty(n, dtype=odt, device=x.device) if out is None else out
    L = load()
    ws = ws if ws is not None else workspace(L.scan_shard_workspace_bytes(dt, n), x.device, stream)
    _check(L.scan_shard_scan_peers(_ptr(x), _ptr(out), n, dt, int(bool(exclusive)), _ptr(slots), G, rank, epoch,
                                   ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)), "scan_shard_scan_peers")
    return out


def widen_copy(x: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """Measurement ceiling: out = widen(x), the scan's traffic with no scan arithmetic."""
    dt, _, _ = _prep(x)
    _check(load().scan_widen_copy(_ptr(x), _ptr(out), x.numel(), dt, _stream_ptr(stream)), "scan_widen_copy")
    return out


def launch_count() -> int:
    return int(load().scan_launch_count())


# ---------------------------------------------------------------- operators
# include/scan_ops.h: split / compress (P281-285) and the LSB radix sort (P287).
SCAN_KEY = {torch.int16: 1, torch.float16: 2, torch.int32: 4, torch.float32: 5}
if hasattr(torch, "uint16"):
    SCAN_KEY[torch.uint16] = 0
if hasattr(torch, "uint32"):
    SCAN_KEY[torch.uint32] = 3


def split(x: torch.Tensor, flags: torch.Tensor, compress: bool = False, with_idx: bool = True,
          out=None, idx_out=None, stream=None):
    """P281-283 SplitInd: stable split, flag-true items first (nonzero int8 = true).

    Returns (z, idx, count) with count a 1-element int64 CUDA tensor (T, the
    number of true flags).  With compress=True (P285, = masked_select) only
    the first T entries of z / idx are meaningful; see compress()."""
    if not (x.is_cuda and flags.is_cuda):
        raise ScanError("split expects CUDA tensors (there is no CPU path)")
    if flags.dtype != torch.int8:
        raise ScanError("flags must be int8")
    x = x.reshape(-1)
    flags = flags.reshape(-1)
    if not (x.is_contiguous() and flags.is_contiguous()) or flags.numel() != x.numel():
        raise ScanError("x and flags must be contiguous 1-D tensors of the same length")
    n = x.numel()
    z = torch.empty_like(x) if out is None else out
    idx = (torch.empty(n, dtype=torch.int32, device=x.device) if idx_out is None else idx_out) \
        if with_idx else None
    cnt = torch.empty(1, dtype=torch.int64, device=x.device)
    L = load()
    ws = workspace(L.scan_split_workspace_bytes(n), x.device, stream, kind="ops")
    _check(L.scan_split(_ptr(x), _ptr(flags), _ptr(z), _ptr(idx), n, x.element_size(), int(bool(compress)),
                        _ptr(cnt), ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)), "scan_split")
    return z, idx, cnt


def compress(x: torch.Tensor, flags: torch.Tensor, with_idx: bool = False, stream=None):
    """P285 compress (= torch.masked_select): the flag-true items of x in order.
    Synchronises once to size the result."""
    z, idx, cnt = split(x, flags, compress=True, with_idx=with_idx, stream=stream)
    T = int(cnt.item())
    return (z[:T], idx[:T]) if with_idx else z[:T]


def radix_sort(keys: torch.Tensor, descending: bool = False, out=None, idx_out=None, stream=None):
    """P286-287 stable LSB radix sort by one split per key bit (16 for 16-bit
    keys, 32 for 32-bit); floats ordered by the IEEE total order (R13).

    Returns (sorted keys, int32 input positions)."""
    if not keys.is_cuda:
        raise ScanError("radix_sort expects a CUDA tensor (there is no CPU path)")
    if keys.dtype not in SCAN_KEY:
        raise ScanError(f"unsupported key dtype {keys.dtype}")
    keys = keys.reshape(-1).contiguous()
    n = keys.numel()
    kout = torch.empty_like(keys) if out is None else out
    idx = torch.empty(n, dtype=torch.int32, device=keys.device) if idx_out is None else idx_out
    L = load()
    kt = SCAN_KEY[keys.dtype]
    ws = workspace(L.scan_radix_sort_workspace_bytes(n, kt), keys.device, stream, kind="ops")
    _check(L.scan_radix_sort(_ptr(keys), _ptr(kout), _ptr(idx), n, kt, int(bool(descending)),
                             ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)), "scan_radix_sort")
    return kout, idx


def radix_sort_rows(keys: torch.Tensor, descending: bool = False, out=None, idx_out=None, stream=None):
    """Sort every row of a 2-D CUDA tensor on its own (the row-batched LSB radix
    sort, scan_radix_sort_rows).  Returns (sorted rows, int32 column indices)."""
    if not keys.is_cuda:
        raise ScanError("radix_sort_rows expects a CUDA tensor (there is no CPU path)")
    if keys.dtype not in SCAN_KEY or keys.dim() != 2:
        raise ScanError("radix_sort_rows expects a 2-D tensor of a supported key dtype")
    keys = keys.contiguous()
    R, C = keys.shape
    kout = torch.empty_like(keys) if out is None else out
    idx = torch.empty((R, C), dtype=torch.int32, device=keys.device) if idx_out is None else idx_out
    L = load()
    kt = SCAN_KEY[keys.dtype]
    ws = workspace(L.scan_radix_sort_rows_workspace_bytes(R, C, kt), keys.device, stream, kind="ops")
    _check(L.scan_radix_sort_rows(_ptr(keys), _ptr(kout), _ptr(idx), R, C, kt, int(bool(descending)),
                                  ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream)), "scan_radix_sort_rows")
    return kout, idx


def weighted_sample(w: torch.Tensor, theta: float, cdf=None, stream=None) -> torch.Tensor:
    """P463 weighted sampling: scan w (fp32, our scan) and draw the index whose
    cumulative interval contains theta * sum(w) (R14).  Returns a 1-element
    int64 CUDA tensor; `cdf` (optional, [n] fp32) receives the scan."""
    if not w.is_cuda or w.dtype != torch.float32:
        raise ScanError("weights must be a CUDA float32 tensor (there is no CPU path)")
    w = w.reshape(-1).contiguous()
    n = w.numel()
    cdf = torch.empty_like(w) if cdf is None else cdf
    out = torch.empty(1, dtype=torch.int64, device=w.device)
    L = load()
    ws = workspace(L.scan_workspace_bytes(SCAN_F32_F32, n), w.device, stream)
    _check(L.scan_weighted_sample(_ptr(w), n, float(theta), _ptr(out), _ptr(cdf), ctypes.c_void_p(ws.ptr),
                                  ws.nbytes, _stream_ptr(stream)), "scan_weighted_sample")
    return out


def top_p_sample(probs: torch.Tensor, p: float, u: torch.Tensor, stream=None, method: str = "select"):
    """P298-299 top-p (nucleus) sampling of every row of `probs` [rows, cols].

    method="select" (default): no full sort -- per row the candidates
    {q >= tau} are sorted in shared memory and scanned (scan_top_p_sample);
    rows that need more than 8192 candidates fall back to the sort path.
    method="sort": the paper's pipeline -- descending stable row sort (our
    row-batched radix sort, scan_radix_sort_rows), our row scan (scan_rows,
    P437) of the sorted probabilities, our nucleus + inverse transform draw
    (scan_top_p_draw, R15).  No library kernel on either path.

    Returns (tokens int64 [rows], nucleus sizes int32 [rows])."""
    if not (probs.is_cuda and u.is_cuda) or probs.dtype != torch.float32 or u.dtype != torch.float32:
        raise ScanError("probs and u must be CUDA float32 tensors (there is no CPU path)")
    if probs.dim() != 2 or u.numel() != probs.shape[0] or (probs.shape[1] > 1 and probs.stride(1) != 1):
        raise ScanError("probs must be [rows, cols] with unit column stride and u [rows]")
    R, C = probs.shape
    u = u.contiguous()
    tok = torch.empty(R, dtype=torch.int64, device=probs.device)
    kept = torch.empty(R, dtype=torch.int32, device=probs.device)
    if method == "select":
        ws = workspace(0, probs.device, stream, kind="ops")
        _check(load().scan_top_p_sample(_ptr(probs), R, C, probs.stride(0) if R > 1 else C, float(p), _ptr(u),
                                        _ptr(tok), _ptr(kept), ctypes.c_void_p(ws.ptr), ws.nbytes,
                                        _stream_ptr(stream)), "scan_top_p_sample")
        miss = torch.nonzero(tok < 0).flatten()
        if miss.numel() == 0:
            return tok, kept
        t2, k2 = top_p_sample(probs[miss], p, u[miss], stream=stream, method="sort")
        tok[miss] = t2
        kept[miss] = k2
        return tok, kept
    sp, order = radix_sort_rows(probs, descending=True, stream=stream)
    cdf = rows(sp, stream=stream)
    _check(load().scan_top_p_draw(_ptr(cdf), _ptr(order), R, C, cdf.stride(0), order.stride(0), float(p),
                                  _ptr(u), _ptr(tok), _ptr(kept), _stream_ptr(stream)),
           "scan_top_p_draw")
    return tok, kept
