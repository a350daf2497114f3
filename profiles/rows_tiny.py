"""Strided tiny-row scans (rows of <= 32 columns at a wider row stride): CUDA-event time per
scan_rows call, median of 10, for a few shapes (profiles/r02c_rows_tiny.txt).
    [SCAN_LIB=...] [SCAN_ROWS_TILE_STRIDED=0] python profiles/rows_tiny.py
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_15112_b200 as S
lib = os.environ.get("SCAN_LIB", "libscan.so")
for dt, R, C, Sd in [(torch.float32, 1 << 20, 32, 48), (torch.float32, 1 << 21, 16, 24), (torch.int32, 1 << 20, 32, 64), (torch.float16, 1 << 21, 32, 48), (torch.float32, 1 << 22, 8, 16)]:
    X = torch.randn(R, Sd, device="cuda").to(dt)[:, :C] if dt != torch.int32 else torch.randint(-100, 100, (R, Sd), device="cuda", dtype=torch.int32)[:, :C]
    out = torch.empty(R, C, device="cuda", dtype=torch.int32 if dt == torch.int32 else torch.float32)
    for _ in range(3): S.rows(X, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); S.rows(X, out=out); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); ms = ts[5]
    alg = R * C * (X.element_size() + 4)
    print(f"{lib} {dt} {R}x{C} stride {Sd}: {ms*1e3:.1f} us, {alg/ms/1e6:.0f} GB/s alg ({100*alg/ms/1e6/6549.4:.1f} %)")
