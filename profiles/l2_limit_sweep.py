"""C5 / C2 / C3 scan rate against cudaLimitPersistingL2CacheSize (the L2 set-aside
that evict_last lines may occupy).  One process, one box; the same inputs for every
setting; alternated twice.

    python profiles/l2_limit_sweep.py [C5 C2 C3]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

LIMIT = 0x06  # cudaLimitPersistingL2CacheSize


def main():
    cfgs = sys.argv[1:] or ["C5"]
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    rt = ctypes.CDLL("libcudart.so.12")
    cur = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(cur), LIMIT)
    default = cur.value
    print("default limit bytes", default, flush=True)
    for cfg in cfgs:
        run = bench.Run(cfg, 0, 1, torch.device("cuda", 0))
        for rep in range(2):
            for mb in (None, 0, 4, 8, 16, 48):
                val = default if mb is None else mb << 20
                rc = -1
                if not os.environ.get("NOSET"):
                    rc = rt.cudaDeviceSetLimit(LIMIT, ctypes.c_size_t(val))
                rt.cudaDeviceGetLimit(ctypes.byref(cur), LIMIT)
                m = run.measure(10, 3, True, lambda: None)
                print(f"{cfg} limit={'default' if mb is None else mb} rc={rc} now={cur.value} "
                      f"ms={m['ms_per_step']:.4f} frac={m['roof']['frac']}", flush=True)
        if not os.environ.get("NOSET"):
            rt.cudaDeviceSetLimit(LIMIT, ctypes.c_size_t(default))
        del run
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
