# Runner for the tensor-core A/B ncu capture (profiles/r01_tc_ab_rows.txt):
#   ncu --set full -k regex:k_rowscan -s 1 -c 4 python profiles/run_tc_ab.py
# Rows 32768 x 16384 of fp16 -> fp32 and int8 -> int32: SCAN_ROWS_TC=0 (CUDA-core
# k_rowscan16) then =1 (tcgen05 k_rowscan_tc, kind::f16 / kind::i8).
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

R, C = 32768, 16384
for dt, kind, seed in ((torch.float16, inputs.F16_U01, 1), (torch.int8, inputs.I8_FLAG, 2)):
    x = torch.empty(R * C, dtype=dt, device="cuda")
    inputs.fill_device(kind, seed, 0, R * C, 0, x)
    x = x.view(R, C)
    o = torch.empty(R, C, dtype=torch.int32 if dt == torch.int8 else torch.float32, device="cuda")
    for tc in ("0", "1"):
        os.environ["SCAN_ROWS_TC"] = tc
        for _ in range(2):
            S.rows(x, out=o)
    torch.cuda.synchronize()
    del x, o
