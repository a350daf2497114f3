"""Minimal runner for ncu captures: fills one config's input on cuda:0 and runs
the 1-D scan `reps` times through the C ABI binding (no timing, no oracle).

    ncu --set full --clock-control none --import-source on -k regex:k_mcscan16 \
        -s 2 -c 1 -o r01_C5_full python profiles/run_scan.py C5 3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

SPEC = {  # config: (input dtype, n, recipe, seed, exclusive)
    "C2": (torch.float16, 1 << 28, inputs.F16_U01, 1, False),
    "C3": (torch.int8, 1 << 30, inputs.I8_FLAG, 2, True),
    "C5": (torch.float32, 1 << 32, inputs.F32_NORMAL, 4, False),
}

if __name__ == "__main__":
    cfg = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dt, n, kind, seed, exc = SPEC[cfg]
    x = torch.empty(n, dtype=dt, device="cuda")
    inputs.fill_device(kind, seed, 0, n, 0, x)
    out = torch.empty(n, dtype=torch.int32 if dt == torch.int8 else torch.float32, device="cuda")
    for _ in range(reps):
        (S.exclusive if exc else S.inclusive)(x, out=out)
    torch.cuda.synchronize()
    print("done", cfg)
