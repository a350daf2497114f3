"""Does a plain copy keep the burst rate under sustained load?  torch copy_ of 16 GiB
(32 GiB of traffic per iteration, C5's bytes) and cudaMemcpyAsync-free widen copy
(libscan's scan_widen_copy on the same arrays), 80 iterations each after 0.5 s idle;
per-iteration CUDA-event times, then the C5 scan the same way.

    python profiles/copy_sustained.py
"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402


def series(fn, n=80):
    stream = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    time.sleep(0.5)
    evs = []
    for i in range(n + 1):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        evs.append(e)
        if i < n:
            fn()
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw", "--format=csv,noheader"],
                       capture_output=True, text=True).stdout.strip()
    torch.cuda.synchronize()
    return [evs[i].elapsed_time(evs[i + 1]) for i in range(n)], q


def main():
    torch.cuda.set_device(0)
    run = bench.Run("C5", 0, 1, torch.device("cuda", 0))
    x, out = run.x, run.out
    nbytes = 2 * x.numel() * 4
    for name, fn in (("torch copy_", lambda: out.copy_(x)),
                     ("C5 scan", run.step),
                     ("torch copy_", lambda: out.copy_(x)),
                     ("C5 scan", run.step)):
        ts, q = series(fn)
        first, last = sum(ts[1:7]) / 6, sum(ts[-20:]) / 20
        print(f"{name}: first 6 {first:.3f} ms ({nbytes / first / 1e6:.0f} GB/s), last 20 {last:.3f} ms "
              f"({nbytes / last / 1e6:.0f} GB/s); smi under load: {q}", flush=True)
        print("   ", " ".join(f"{t:.2f}" for t in ts), flush=True)


if __name__ == "__main__":
    main()
