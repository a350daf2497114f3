"""Launch / fill / drain timeline of one k_mcscan16 launch from the per-CTA
globaltimer stamps of the profiling build (-DSCAN_MC_PROF: mcscan.cuh s_prof[21..24]
= entry, first tile in (compute warp 0), compute warp 0 done, exit).

    SCAN_LIB=libscan_prof.so SCAN_DEBUG=4 python profiles/mc_timeline.py C2 [log2 n]

Also prints the back-to-back CUDA-event time per launch of the same scan (10 launches),
so the in-kernel spans can be set against the per-launch cost.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

SPEC = {"C2": (torch.float16, 28, inputs.F16_U01, 1, False, 6),
        "C3": (torch.int8, 30, inputs.I8_FLAG, 2, True, 5),
        "C5": (torch.float32, 32, inputs.F32_NORMAL, 4, False, 8)}
NPROF = 25
KWS_PARTIALS = 256


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    dt, lg, kind, seed, exc, bpe = SPEC[cfg]
    if len(sys.argv) > 2:
        lg = int(sys.argv[2])
    n = 1 << lg
    x = torch.empty(n, dtype=dt, device="cuda")
    inputs.fill_device(kind, seed, 0, n, 0, x)
    out = torch.empty(n, dtype=torch.int32 if dt == torch.int8 else torch.float32, device="cuda")
    fn = S.exclusive if exc else S.inclusive
    for _ in range(3):
        fn(x, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fn(x, out=out)
    b.record()
    torch.cuda.synchronize()
    per = a.elapsed_time(b) / 10 * 1e3
    fn(x, out=out)
    torch.cuda.synchronize()
    ws = S.workspace(0, x.device)
    nct = torch.cuda.get_device_properties(0).multi_processor_count
    off = ws.ptr - ws.buf.data_ptr() + KWS_PARTIALS
    v = ws.buf[off:off + nct * NPROF * 8].clone().view(torch.int64).view(nct, NPROF).cpu().double()
    ent, first, cdone, ex = v[:, 21], v[:, 22], v[:, 23], v[:, 24]
    t0 = ent.min()
    us = lambda t: (t - t0) / 1e3  # noqa: E731
    print(f"{cfg} n=2^{lg}: back-to-back {per:.1f} us per launch ({n * bpe / per / 1e3:.0f} GB/s); "
          f"kernel span (first entry -> last exit) {us(ex.max()):.1f} us")
    print(f"  entry: last CTA {us(ent.max()):.2f} us after the first")
    print(f"  first tile in (compute warp 0): min {us(first.min()):.2f} median {us(first.median()):.2f} "
          f"max {us(first.max()):.2f} us")
    print(f"  compute warp 0 done: min {us(cdone.min()):.1f} median {us(cdone.median()):.1f} max {us(cdone.max()):.1f} us")
    print(f"  exit: min {us(ex.min()):.1f} median {us(ex.median()):.1f} max {us(ex.max()):.1f} us")
    if os.environ.get("MC_TIMELINE_DUMP"):
        for i in range(nct):
            print(i, f"{us(ent[i]):.2f} {us(first[i]):.2f} {us(cdone[i]):.1f} {us(ex[i]):.1f}")


if __name__ == "__main__":
    main()
