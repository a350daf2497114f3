"""Top-p select kernel timing on the C4 rows (4096 x 131072 softmax(4 N(0,1)), p = 0.9):
CUDA events around scan_top_p_sample, median of `reps`.  Run once plain and once with
SCAN_TOPP_DBG=1 (every row stops after the candidate pass) to split pass / rest.

    [SCAN_TOPP_DBG=1] python profiles/topp_phase.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    R, C = 4096, 131072
    probs = torch.empty((R, C), dtype=torch.float32, device="cuda")
    inputs.fill_device(inputs.F32_SOFTMAX, 3, 0, R, C, probs)
    uu = torch.rand(R, generator=torch.Generator(device="cuda").manual_seed(7), device="cuda")
    for _ in range(3):
        tok, kept = S.top_p_sample(probs, 0.9, uu)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.top_p_sample(probs, 0.9, uu)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SCAN_TOPP"))
    extra = ""
    if os.environ.get("SCAN_TOPP_DBG") == "1":
        extra = (f", candidates per row: mean {tok.double().mean().item():.0f} max {tok.max().item()}, "
                 f"rows over 8192 (superset overflow -> re-read fallback): {(tok > 8192).sum().item()}")
    if os.environ.get("SCAN_TOPP_DBG") == "5":
        codes = (-10 - tok[tok <= -10]).cpu()
        extra = (f", rows the level path did not finish: {codes.numel()}, by cause (0 other, 1 overflow, "
                 f"2 short mass, 3 big level): {torch.bincount(codes, minlength=4).tolist()}")
    print(f"top-p select {env or '(default)'}: {ms:.4f} ms median of {reps}, "
          f"{R * C * 4 / ms / 1e6:.1f} GB/s of rows{extra}")


if __name__ == "__main__":
    main()
