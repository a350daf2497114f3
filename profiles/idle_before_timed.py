"""Does the 0.3 s idle before the timed region (the clock sampler's start) change the
C5 number?  Same process, same arrays, alternating; also longer timed regions.

    python profiles/idle_before_timed.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    torch.cuda.set_device(0)
    run = bench.Run(cfg, 0, 1, torch.device("cuda", 0))
    for rep in range(3):
        for steps, sampler in ((10, True), (10, False), (40, True), (40, False), (100, True)):
            m = run.measure(steps, 3, True, lambda: None, clocks=bench.ClockSampler(0) if sampler else None)
            print(f"{cfg} steps={steps} idle_0.3s={sampler} ms={m['ms_per_step']:.4f} frac={m['roof']['frac']} "
                  f"clocks={m['clocks']}", flush=True)
    # eager per-step times of a long run: where does the rate change?
    stream = torch.cuda.current_stream()
    time.sleep(0.5)
    evs = []
    for i in range(61):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        evs.append(e)
        if i < 60:
            run.step()
    torch.cuda.synchronize()
    print("eager per-step ms after 0.5 s idle:",
          " ".join(f"{evs[i].elapsed_time(evs[i + 1]):.2f}" for i in range(60)), flush=True)


if __name__ == "__main__":
    main()
