"""Per-GPU work of the sharded (multi-GPU) scan, timed on ONE B200, and the
aggregate it projects to at G GPUs (weak in work per GPU, strong in n).

Each "rank" of a G-way split of C5 (fp32, n = 2^32) / C3 (int8 -> int32
exclusive, n = 2^30) does, on its own shard:
  new:  scan_shard_reduce (one read) + carry_from_totals + scan_shard_scan
        (row-kernel stream with per-block starts)       [paper_2505_15112_b200.dist]
  old:  scan_total (one read) + carry_from_totals + scan with carry (MCScan)
The NCCL all-gather of G x 8 bytes is not included (NVLink latency, ~10-20 us);
rss_peer_exchange has no all-gather at all (the totals travel inside the two
kernels), its slot writes here are local (emulated peers) -- over NVLink each
rank's publish adds G remote 16-byte stores.
CUDA events, median of 5 single calls after 2 warm-ups (per_gpu_us: includes the
host launch latency of every call) and the per-call time of 10 calls replayed from one
CUDA graph (graph_per_gpu_us: the device's back-to-back rate); rank 1's shard
(nonzero carry).

    python profiles/shard_projection.py [C5|C3 ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402
from bench import peaks  # noqa: E402

CFG = {"C5": (torch.float32, 1 << 32, inputs.F32_NORMAL, 4, False, 8),
       "C3": (torch.int8, 1 << 30, inputs.I8_FLAG, 2, True, 5)}


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def timed_graph(fn, reps=10):
    """Per-call time of `reps` calls captured back to back in one CUDA graph
    (the device's back-to-back rate, without per-call host launch latency)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3 / reps)
    del g
    return min(ts)


def main():
    peak, _ = peaks()
    out = []
    for cfg in (sys.argv[1:] or ["C5", "C3"]):
        dt, n, kind, seed, exc, bpe = CFG[cfg]
        for G in (1, 2, 4, 8):
            m = n // G
            x = torch.empty(m, dtype=dt, device="cuda")
            inputs.fill_device(kind, seed, m, m, 0, x)  # rank 1's shard
            y = torch.empty(m, dtype=torch.int32 if dt == torch.int8 else torch.float32, device="cuda")
            cdt = torch.int64 if dt == torch.int8 else torch.float64
            totals = torch.ones(G, dtype=cdt, device="cuda")
            ws = S.shard_workspace(x)

            def new():
                S.shard_reduce(x, ws=ws)
                c = S.carry_from_totals(totals, min(1, G - 1), dt)
                S.shard_scan(x, exc, carry_in=c, ws=ws, out=y)

            def old():
                S.total(x)
                c = S.carry_from_totals(totals, min(1, G - 1), dt)
                (S.exclusive if exc else S.inclusive)(x, out=y, carry_in=c)

            def single():
                (S.exclusive if exc else S.inclusive)(x, out=y)

            # device-initiated exchange: rank 1 of G, the lower rank's slot
            # pre-published (emulated peers: all slot arrays on this GPU)
            Gp = max(G, 2)
            slots = [torch.zeros(S.peer_slots_bytes(Gp) // 8, dtype=torch.int64, device="cuda") for _ in range(Gp)]
            peers = torch.tensor([t.data_ptr() for t in slots], dtype=torch.int64, device="cuda")
            x0 = torch.zeros(1, dtype=dt, device="cuda")
            ws0 = S.shard_workspace(x0)
            ep = [0]

            def peer():
                ep[0] += 1
                S.shard_reduce_publish(x0, peers.data_ptr(), Gp, 0, ep[0], ws=ws0)  # rank 0 (1 element)
                S.shard_reduce_publish(x, peers.data_ptr(), Gp, 1, ep[0], ws=ws)
                S.shard_scan_peers(x, exc, slots[1], Gp, 1, ep[0], ws=ws, out=y)

            rec = {"config": cfg, "G": G, "shard_elems": m}
            for name, fn in (("rss_blocks", new), ("rss_peer_exchange", peer), ("rss_mcscan", old),
                             ("single_pass", single)):
                t = timed(fn)
                tg = timed_graph(fn)
                rec[name] = {"per_gpu_us": round(t * 1e6, 1), "per_gpu_pct_alg": round(100 * m * bpe / t / 1e9 / peak, 1),
                             "aggregate_GBps": round(G * m * bpe / t / 1e9, 0),
                             "graph_per_gpu_us": round(tg * 1e6, 1),
                             "graph_per_gpu_pct_alg": round(100 * m * bpe / tg / 1e9 / peak, 1)}
            print(json.dumps(rec), flush=True)
            out.append(rec)
            del x, y, ws
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
