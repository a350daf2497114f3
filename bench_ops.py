#!/usr/bin/env python
"""bench_ops.py -- the scan-based operators of PAPER.md Sec. 5 on one B200
(SURVEY.md 8(f) rows): split / SplitInd (P281-283), compress (P285, vs
torch.masked_select), the LSB radix sort by per-bit splits (P286-287, vs
torch.sort), weighted sampling (P463) and top-p sampling (P298-299).

    python bench_ops.py --op split|compress|sort|weighted|top_p [--steps K] [--warmup W]

Prints one JSON line in the shape of bench.py's (metric GB/s of algorithmic
bytes, roofline against the measured HBM peak, cpu_baseline = the oracle as
it stands on a bounded sample, clocks), plus the torch library routine timed
on the same input as context.  Inputs are seeded and synthetic (inputs/).
bench.py (the driver's line, C5) is unaffected.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from bench import ClockSampler, log, peaks  # noqa: E402

OPS = {
    "split": dict(name="SplitInd: fp16 payload + int32 indices, C3 mask (n=2^30, Bernoulli 0.5, seed 2)",
                  n=1 << 30),
    "compress": dict(name="compress (masked_select): fp16 payload, C3 mask (n=2^30, Bernoulli 0.5, seed 2)",
                     n=1 << 30),
    "sort": dict(name="LSB radix sort (8-bit digits, 2 passes; SCAN_SORT_BITS=1: the paper's 16 splits): "
                      "fp16 keys N(0,1) + int32 indices, n=2^24, seed 5",
                 n=1 << 24),
    "weighted": dict(name="weighted sampling: scan of n=2^28 fp32 weights U[0,1) (seed 6) + one draw",
                     n=1 << 28),
    "top_p": dict(name="top-p sampling: 4096 rows x 131072 softmax(4*N(0,1)) fp32 (C4 rows), p=0.9, "
                       "row sort + row scan + nucleus draw", n=4096 * 131072),
    "sort_rows": dict(name="row-batched LSB radix sort, descending stable: 4096 rows x 131072 softmax(4*N(0,1)) "
                           "fp32 (C4 rows) + int32 column indices (the top-p sort path's sort)", n=4096 * 131072),
}


def time_events(fn, steps, warmup, stream):
    import torch
    for _ in range(warmup):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    for i in range(steps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(steps)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", choices=sorted(OPS), default="split")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--top-p-method", choices=["select", "sort"], default="select")
    args = ap.parse_args()
    import numpy as np
    import torch

    import inputs
    import paper_2505_15112_b200 as S
    S.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    w = OPS[args.op]
    n = w["n"]
    peak, peak_src = peaks()
    launches0 = S.launch_count()

    if args.op in ("split", "compress"):
        f = torch.empty(n, dtype=torch.int8, device=dev)
        inputs.fill_device(inputs.I8_FLAG, 2, 0, n, 0, f)
        x = torch.empty(n, dtype=torch.float16, device=dev)
        inputs.fill_device(inputs.F16_U01, 1, 0, n, 0, x)
        z = torch.empty_like(x)
        idx = torch.empty(n, dtype=torch.int32, device=dev)
        T = int(f.sum(dtype=torch.int64).item())
        if args.op == "split":
            fn = lambda: S.split(x, f, out=z, idx_out=idx)  # noqa: E731
            alg = n * (1 + 2 + 2 + 4)
        else:
            fn = lambda: S.split(x, f, compress=True, with_idx=False, out=z)  # noqa: E731
            alg = n * (1 + 2) + T * 2
        fb = f.bool()
        ref_fn = lambda: torch.masked_select(x, fb)  # noqa: E731
        ref_name = "torch.masked_select (bool mask)"
    elif args.op == "sort":
        k = torch.empty(n, dtype=torch.float32, device=dev)
        inputs.fill_device(inputs.F32_NORMAL, 5, 0, n, 0, k)
        k = k.half()
        ko = torch.empty_like(k)
        idx = torch.empty(n, dtype=torch.int32, device=dev)
        fn = lambda: S.radix_sort(k, out=ko, idx_out=idx)  # noqa: E731
        # 8-bit digits: 2 passes, each keys in + out and indices in + out (pass 0 reads none)
        passes = 16 if os.environ.get("SCAN_SORT_BITS") == "1" else 2
        alg = passes * n * (2 + 2 + 4 + 4) - n * 4
        ref_fn = lambda: torch.sort(k, stable=True)  # noqa: E731
        ref_name = "torch.sort(stable=True) (CUB radix sort, int64 indices)"
    elif args.op == "sort_rows":
        R, C = 4096, 131072
        k = torch.empty((R, C), dtype=torch.float32, device=dev)
        inputs.fill_device(inputs.F32_SOFTMAX, 3, 0, R, C, k)
        ko = torch.empty_like(k)
        idx = torch.empty((R, C), dtype=torch.int32, device=dev)
        fn = lambda: S.radix_sort_rows(k, descending=True, out=ko, idx_out=idx)  # noqa: E731
        # 4 passes of 8-bit digits: keys in + out, indices in + out (pass 0 reads none)
        alg = 4 * n * (4 + 4 + 4 + 4) - n * 4
        ref_fn = lambda: torch.sort(k, dim=1, descending=True, stable=True)  # noqa: E731
        ref_name = "torch.sort(dim=1, descending=True, stable=True) (CUB segmented sort, int64 indices)"
    elif args.op == "weighted":
        wgt = torch.empty(n, dtype=torch.float32, device=dev)
        inputs.fill_device(inputs.F32_NORMAL, 6, 0, n, 0, wgt)
        wgt = wgt.abs_()
        cdf = torch.empty_like(wgt)
        fn = lambda: S.weighted_sample(wgt, 0.37, cdf=cdf)  # noqa: E731
        alg = n * 8  # the scan's in + out; the draw probes O(1) KB
        ref_fn = lambda: torch.searchsorted(torch.cumsum(wgt, 0), 0.37 * wgt.sum(), right=True)  # noqa: E731
        ref_name = "torch.cumsum + torch.searchsorted (torch.multinomial caps categories at 2^24)"
    else:  # top_p
        R, C = 4096, 131072
        probs = torch.empty((R, C), dtype=torch.float32, device=dev)
        inputs.fill_device(inputs.F32_SOFTMAX, 3, 0, R, C, probs)
        uu = torch.rand(R, generator=torch.Generator(device=dev).manual_seed(7), device=dev)
        fn = lambda: S.top_p_sample(probs, 0.9, uu, method=args.top_p_method)  # noqa: E731
        alg = R * C * 4  # bytes of probabilities consumed per step

        def ref_fn():
            sp, order = torch.sort(probs, dim=1, descending=True, stable=True)
            cs = torch.cumsum(sp, dim=1)
            keep = (cs - sp) < 0.9
            sp = sp * keep
            tok = torch.searchsorted(torch.cumsum(sp, 1), (uu * sp.sum(1)).unsqueeze(1), right=True)
            return order.gather(1, tok.clamp_max(C - 1))
        ref_name = "torch.sort + torch.cumsum + mask + searchsorted (Llama-style top-p)"

    clocks = ClockSampler(0)
    clocks.start()
    times = time_events(fn, args.steps, args.warmup, stream)
    clk = clocks.stop()
    launches = (S.launch_count() - launches0) * args.steps // (args.steps + args.warmup)
    ref_times = time_events(ref_fn, max(3, args.steps // 2), 2, stream)
    med = statistics.median(times)
    value = alg / med / 1e9

    # cpu_baseline: the oracle as it stands on a bounded sample of the same workload
    import oracle
    cn = 1 << 22 if args.op not in ("sort", "sort_rows") else 1 << 18
    if args.op == "sort_rows":
        cn = 131072
        Ph = inputs.fill_host(inputs.F32_SOFTMAX, 3, 0, 1, cn)[0]
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            oracle.radix_sort(Ph, "f32", descending=True)
            reps += 1
        ct = time.perf_counter() - t0
        cpu_alg = alg / n * cn * reps
    elif args.op == "top_p":
        cn = 131072
        Ph = inputs.fill_host(inputs.F32_SOFTMAX, 3, 0, 1, C)[0]
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            oracle.top_p_sample(Ph, 0.9, 0.5)
            reps += 1
        ct = time.perf_counter() - t0
        cpu_alg = cn * 4 * reps
    elif args.op == "weighted":
        wh = np.abs(inputs.fill_host(inputs.F32_NORMAL, 6, 0, cn))
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            oracle.weighted_sample(wh, 0.37)
            reps += 1
        ct = time.perf_counter() - t0
        cpu_alg = cn * 8 * reps
    elif args.op in ("split", "compress"):
        fh = inputs.fill_host(inputs.I8_FLAG, 2, 0, cn)
        xh = inputs.fill_host(inputs.F16_U01, 1, 0, cn)
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            oracle.split(xh, fh, compress=args.op == "compress", with_idx=args.op == "split")
            reps += 1
        ct = time.perf_counter() - t0
        cpu_alg = alg / n * cn * reps
    else:
        kh = np.random.default_rng(5).standard_normal(cn).astype(np.float16)
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            oracle.radix_sort(kh, "f16")
            reps += 1
        ct = time.perf_counter() - t0
        cpu_alg = alg / n * cn * reps
    line = {
        "metric": f"{args.op} GB/s (algorithmic bytes)", "value": round(value, 1), "unit": "GB/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(med * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"split": "fp16 payload / int8 mask / int32 indices", "compress": "fp16 payload / int8 mask",
                  "sort": "fp16 keys / int32 indices", "weighted": "f32 (fp64 carry)",
                  "top_p": "f32 probabilities / int64 tokens",
                  "sort_rows": "f32 keys / int32 column indices"}[args.op],
        "data": "synthetic (seeded counter-based generator, inputs/recipe.h; generated in HBM)",
        "config": {"workload": w["name"] + (f" [method={args.top_p_method}]" if args.op == "top_p" else ""),
                   "n_elements": n, "alg_bytes_per_step": alg,
                   "gelem_per_s": round(n / med / 1e9, 2),
                   "l2_flush": "not needed: inputs exceed the 126 MB L2"},
        "roofline": {"bound": "hbm", "achieved": round(value, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(value / peak, 4), "traffic": None, "peak_source": peak_src},
        "cpu_baseline": {"value": round(cpu_alg / ct / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{reps} x {cn} elements of the same recipe, single-thread C oracle"},
        "library_baseline": {"name": ref_name, "ms": round(statistics.median(ref_times) * 1e3, 4),
                             "speedup": round(statistics.median(ref_times) / med, 3)},
        "gpu_launches": launches, "clocks": clk,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
