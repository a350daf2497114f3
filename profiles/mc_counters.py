"""Per-CTA stall counters of k_mcscan16 (SCAN_DEBUG=4) plus a CUDA-event timing,
for one config under the current SCAN_MC_* environment.

    SCAN_MC_BT=1 SCAN_MC_AHEAD=3 [SCAN_DEBUG=4] python profiles/mc_counters.py C5

The counters are the kernel's own clock64() sums (mcscan.cuh, s_prof), copied
into the workspace's partials area at kernel end.  The timed runs are separate
from the counter run: run the script once without SCAN_DEBUG (timing) and once with
SCAN_DEBUG=4 (counters of the last call; its timing includes the counters' clock reads).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

SPEC = {  # config: (input dtype, n, recipe, seed, exclusive, bytes per element in+out)
    "C2": (torch.float16, 1 << 28, inputs.F16_U01, 1, False, 6),
    "C3": (torch.int8, 1 << 30, inputs.I8_FLAG, 2, True, 5),
    "C5": (torch.float32, 1 << 32, inputs.F32_NORMAL, 4, False, 8),
}
NAMES = ["c_wait_carry", "c_wait_in_R", "c_wait_in_S", "c_wait_out_empty", "coord_spin", "storer_wait_ready",
         "storer_bulk_wait", "total", "R_tiles", "S_tiles", "R_cycles", "S_pre", "S_bar", "S_post", "e14", "e15",
         "e16", "e17", "pub_to_complete", "complete_to_sums", "chunks"]
KWS_PARTIALS = 256


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    dt, n, kind, seed, exc, bpe = SPEC[cfg]
    x = torch.empty(n, dtype=dt, device="cuda")
    inputs.fill_device(kind, seed, 0, n, 0, x)
    out = torch.empty(n, dtype=torch.int32 if dt == torch.int8 else torch.float32, device="cuda")
    fn = S.exclusive if exc else S.inclusive
    for _ in range(3):
        fn(x, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(x, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    gbs = n * bpe / ms / 1e6
    env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SCAN_MC"))
    print(f"== {cfg} {env or '(defaults)'}: {ms:.4f} ms median of {reps}, {gbs:.1f} GB/s")
    if os.environ.get("SCAN_DEBUG") != "4":  # the library reads SCAN_DEBUG once per process
        return
    ws = S.workspace(0, x.device)
    nct = torch.cuda.get_device_properties(0).multi_processor_count
    raw = torch.empty(nct * len(NAMES), dtype=torch.int64, device="cuda")
    nbytes = raw.numel() * 8
    buf = ws.buf[ws.ptr - ws.buf.data_ptr() + KWS_PARTIALS:][:nbytes]
    v = buf.clone().view(torch.int64).view(nct, len(NAMES)).double().cpu()
    tot = v[:, 7]
    print(f"total cycles per CTA: min {tot.min():.0f} median {tot.median():.0f} max {tot.max():.0f}")
    for i, nm in enumerate(NAMES):
        if i == 7:
            continue
        c = v[:, i]
        print(f"{nm:18s} mean {c.mean():.3g} ({100 * c.mean() / tot.mean():.1f}% of total) min {c.min():.3g} "
              f"max {c.max():.3g}")
    ch = v[:, 20].mean()
    if ch > 0:
        clk = 1965e6
        print(f"per chunk: publish -> complete {v[:, 18].mean() / ch:.0f} cycles "
              f"({v[:, 18].mean() / ch / clk * 1e6:.2f} us), complete -> sums {v[:, 19].mean() / ch:.0f} cycles; "
              f"chunk period {tot.mean() / ch / clk * 1e6:.2f} us")


if __name__ == "__main__":
    main()
