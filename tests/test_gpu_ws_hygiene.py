"""Workspace / launch hygiene through the C ABI (round-1 advisor findings).

* Operator scratch (split tile counts, radix temporaries) in a workspace that is
  then handed to a look-back scan must not be read as tagged descriptors
  (include/scan.h "Operators ... keep scratch"): scans after split / compress /
  sort on the SAME workspace stay bit-exact against the oracle.
* rows() of an expanded view (row stride < cols) scans a dense copy instead of
  reading past the allocation; an overlapping `out` is refused.
* top-p row tickets live in the caller's workspace: a CUDA-graph replay and
  eager calls interleaved on one stream give the eager results.
"""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ws(cuda, nbytes):
    return cuda.Workspace(nbytes, torch.device("cuda"))


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("op", ["compress", "split", "sort"])
def test_scan_after_operator_on_same_workspace(cuda, oracle, inputs_mod, op):
    L = cuda.load()
    n_op = 1 << 20
    n_scan = 200_000
    need = max(L.scan_split_workspace_bytes(n_op), L.scan_radix_sort_workspace_bytes(n_op, 4),
               L.scan_workspace_bytes(cuda.SCAN_I32_I32, n_scan + 1), L.scan_rows_workspace_bytes(1, 64, 40000))
    ws = _ws(cuda, need)
    rng = np.random.default_rng(5)
    for it in range(12):
        # sparse flags whose per-tile true counts take small values (1..40): the
        # values a fresh workspace's epochs take, the advisor's collision case
        f = np.zeros(n_op, np.int8)
        for t in range(n_op // 8192):
            k = 1 + (t + it) % 40
            f[t * 8192 + rng.choice(8192, k, replace=False)] = 1
        fd = torch.from_numpy(f).cuda()
        x = torch.arange(n_op, dtype=torch.int32, device="cuda")
        z = torch.empty_like(x)
        idx = torch.empty(n_op, dtype=torch.int32, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        if op in ("compress", "split"):
            rc = L.scan_split(_p(x), _p(fd), _p(z), _p(idx), n_op, 4, int(op == "compress"), _p(cnt),
                              ctypes.c_void_p(ws.ptr), ws.nbytes, _stream())
        else:
            keys = torch.from_numpy(rng.integers(0, 1 << 20, n_op, dtype=np.int32)).cuda()
            rc = L.scan_radix_sort(_p(keys), _p(z), _p(idx), n_op, 4, 0, ctypes.c_void_p(ws.ptr), ws.nbytes,
                                   _stream())
        assert rc == 0
        # unaligned 1-D int32 scan > 65,536 elements: the decoupled look-back kernel
        h = inputs_mod.fill_host(inputs_mod.I32_FULL, 100 + it, 0, n_scan + 1)
        xd = torch.from_numpy(h).cuda()[1:]
        out = torch.empty(n_scan + 1, dtype=torch.int32, device="cuda")[1:]
        rc = L.scan_inclusive(_p(xd), _p(out), n_scan, cuda.SCAN_I32_I32, None, ctypes.c_void_p(ws.ptr),
                              ws.nbytes, _stream())
        assert rc == 0
        assert np.array_equal(out.cpu().numpy(), oracle.inclusive(h[1:], "i32")), (op, it)
        # strided rows that take the look-back row path (row stride not 16-byte aligned)
        R, C, S = 64, 40000, 40001
        hr = inputs_mod.fill_host(inputs_mod.I32_FULL, 200 + it, 0, R * S).reshape(R, S)
        Xd = torch.from_numpy(hr).cuda()
        outr = torch.empty((R, C), dtype=torch.int32, device="cuda")
        rc = L.scan_rows(_p(Xd), _p(outr), R, C, S, C, cuda.SCAN_I32_I32, 0, ctypes.c_void_p(ws.ptr), ws.nbytes,
                         _stream())
        assert rc == 0
        assert np.array_equal(outr.cpu().numpy(), oracle.rows(np.ascontiguousarray(hr[:, :C]), "i32")), (op, it)


def test_rows_expanded_view_and_overlapping_out(cuda, oracle, inputs_mod):
    C = 3000
    h = inputs_mod.fill_host(inputs_mod.I32_FULL, 9, 0, C)
    X = torch.from_numpy(h).cuda().expand(64, C)  # stride(0) == 0
    got = cuda.rows(X).cpu().numpy()
    ref = oracle.inclusive(h, "i32")
    assert np.array_equal(got, np.broadcast_to(ref, (64, C)))
    out = torch.empty(C, dtype=torch.int32, device="cuda").expand(64, C)
    with pytest.raises(cuda.ScanError):
        cuda.rows(X, out=out)


def test_top_p_graph_replay_interleaved_with_eager(cuda, inputs_mod):
    L = cuda.load()
    R, C = 64, 131072
    P = torch.from_numpy(inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 0, R, C)).cuda()
    u = torch.from_numpy(np.random.default_rng(3).random(R, dtype=np.float32)).cuda()
    tok_ref, kept_ref = cuda.top_p_sample(P, 0.9, u)
    torch.cuda.synchronize()
    assert bool((tok_ref >= 0).all())
    s = torch.cuda.Stream()
    ws = cuda.workspace(0, torch.device("cuda"), s, kind="ops")
    tok_g = torch.empty(R, dtype=torch.int64, device="cuda")
    kept_g = torch.empty(R, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):  # the C ABI call (the binding's fallback check syncs)
        rc = L.scan_top_p_sample(_p(P), R, C, C, ctypes.c_float(0.9), _p(u), _p(tok_g), _p(kept_g),
                                 ctypes.c_void_p(ws.ptr), ws.nbytes, ctypes.c_void_p(s.cuda_stream))
    assert rc == 0
    for _ in range(70):  # more calls than the old 64-slot ticket ring
        g.replay()
        tok_e, _ = cuda.top_p_sample(P, 0.9, u)
        torch.cuda.synchronize()
        assert torch.equal(tok_g, tok_ref) and torch.equal(kept_g, kept_ref)
        assert torch.equal(tok_e, tok_ref)


def test_scans_inside_cuda_graph(cuda, oracle, inputs_mod):
    """A 1-D MCScan (cooperative persistent launch), an unaligned one (head +
    shifted MCScan) and a row scan captured in ONE CUDA graph and replayed
    several times on fresh inputs: every replay bit-exact (int32)."""
    import torch
    n, R, C = (1 << 22) + 7, 64, 40000
    xs = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    Xr = torch.empty((R, C), dtype=torch.int32, device="cuda")
    y1 = torch.empty(n, dtype=torch.int32, device="cuda")
    y2 = torch.empty(n + 1, dtype=torch.int32, device="cuda")[1:]
    yr = torch.empty((R, C), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm the per-stream workspace outside the capture
        cuda.inclusive(xs[:n], out=y1)
        cuda.exclusive(xs[1:], out=y2)
        cuda.rows(Xr, out=yr)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cuda.inclusive(xs[:n], out=y1)
        cuda.exclusive(xs[1:], out=y2)
        cuda.rows(Xr, out=yr)
    for it in range(3):
        h = inputs_mod.fill_host(inputs_mod.I32_FULL, 40 + it, 0, n + 1)
        hr = inputs_mod.fill_host(inputs_mod.I32_FULL, 50 + it, 0, R * C).reshape(R, C)
        xs.copy_(torch.from_numpy(h))
        Xr.copy_(torch.from_numpy(hr))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(y1.cpu().numpy(), oracle.inclusive(h[:n], "i32")), it
        assert np.array_equal(y2.cpu().numpy(), oracle.exclusive(h[1:], "i32")), it
        assert np.array_equal(yr.cpu().numpy(), oracle.rows(hr, "i32")), it


def test_new_entry_points_reject_bad_arguments(cuda):
    """Argument checks of the round-2 C ABI calls (nothing is launched)."""
    import torch
    L = cuda.load()
    x = torch.zeros(1024, dtype=torch.float32, device="cuda")
    ws = cuda.workspace(1 << 20)
    P = ctypes.c_void_p
    w = P(ws.ptr)
    # row sort: bad key type, cols >= 2^31, workspace too small
    assert L.scan_radix_sort_rows(_p(x), _p(x), _p(x), 4, 256, 9, 0, w, ws.nbytes, _stream()) == 1
    assert L.scan_radix_sort_rows(_p(x), _p(x), _p(x), 1, 1 << 31, 5, 0, w, ws.nbytes, _stream()) == 1
    assert L.scan_radix_sort_rows(_p(x), _p(x), _p(x), 4, 256, 5, 0, w, 16, _stream()) == 2
    # peer exchange: G out of range, rank >= G, epoch 0, NULL slots
    assert L.scan_peer_slots_bytes(0) == 0 and L.scan_peer_slots_bytes(33) == 0
    for G, r, ep, sl in ((0, 0, 1, _p(x)), (4, 4, 1, _p(x)), (4, 1, 0, _p(x)), (4, 1, 1, None)):
        assert L.scan_shard_scan_peers(_p(x), _p(x), 1024, cuda.SCAN_F32_F32, 0, sl, G, r, ep, w, ws.nbytes,
                                       _stream()) == 1
        assert L.scan_shard_reduce_publish(_p(x), 1024, cuda.SCAN_F32_F32, _p(x), sl, G, r, ep, w, ws.nbytes,
                                           _stream()) == 1
    # top-p: workspace required
    assert L.scan_top_p_sample(_p(x), 1, 1024, 1024, ctypes.c_float(0.9), _p(x), _p(x), None, None, 0,
                               _stream()) == 2
