"""Burst vs sustained rate of every config's scan: per-iteration CUDA-event times of
~0.7 s of back-to-back steps (one CUDA-graph replay) after 0.5 s idle.
SCAN_MC_WAIT etc. apply as usual.

    python profiles/sustained_configs.py [C2 C3 C4 C5]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    for cfg in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
        run = bench.Run(cfg, 0, 1, torch.device("cuda", 0))
        for _ in range(3):
            run.step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run.step()
        b.record(stream)
        torch.cuda.synchronize()
        n = max(20, int(1e3 * float(os.environ.get("SUSTAINED_SECONDS", "0.7")) / a.elapsed_time(b)))
        time.sleep(0.5)
        evs = []
        for i in range(n + 1):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append(e)
            if i < n:
                run.step()
        torch.cuda.synchronize()
        ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
        w = bench.WORK[cfg]
        nbytes = run.total_elems * w["bpe"]
        peak = bench.peaks()[0]
        k = max(1, n // 20)
        burst = sorted(ts[1:1 + k])[k // 2]
        sus = sorted(ts[-k:])[k // 2]
        print(f"{cfg}: n={n} burst (median of steps 1..{k}) {burst:.4f} ms = {nbytes / burst / 1e6 / peak:.3f} of peak; "
              f"sustained (median of the last {k}) {sus:.4f} ms = {nbytes / sus / 1e6 / peak:.3f}", flush=True)
        del run
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
