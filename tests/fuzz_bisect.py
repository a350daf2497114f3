"""Run one MCScan-size scan under the fuzz build (SCAN_LIB=libscan_fuzz.so,
SCAN_FUZZ_MASK=sites) and check it; used to bisect a fault-injection failure."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 24) + 7
dt = sys.argv[2] if len(sys.argv) > 2 else "i32"
kind = {"i32": inputs.I32_FULL, "i8": inputs.I8_FULL}[dt]
x = inputs.fill_host(kind, 1, 0, n)
xd = torch.from_numpy(x).cuda()
for exc in (False, True):
    got = (S.exclusive if exc else S.inclusive)(xd).cpu().numpy()
    ref = (oracle.exclusive if exc else oracle.inclusive)(x, dt)
    print("exc" if exc else "inc", "ok" if np.array_equal(got, ref) else "MISMATCH", flush=True)
