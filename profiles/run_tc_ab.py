# Runner for the tensor-core A/B ncu capture (profiles/r01_tc_ab_rows_fp16.txt):
#   ncu --set full -k regex:k_rowscan -s 1 -c 2 python profiles/run_tc_ab.py
# fp16 rows 32768 x 16384: SCAN_ROWS_TC=0 (CUDA-core k_rowscan16) then =1 (tcgen05 k_rowscan_tc).
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, inputs
import paper_2505_15112_b200 as S
R, C = 32768, 16384
x = torch.empty(R * C, dtype=torch.float16, device="cuda"); inputs.fill_device(inputs.F16_U01, 1, 0, R * C, 0, x)
x = x.view(R, C); o = torch.empty(R, C, dtype=torch.float32, device="cuda")
for tc in ("0", "1"):
    os.environ["SCAN_ROWS_TC"] = tc
    for _ in range(2): S.rows(x, out=o)
torch.cuda.synchronize()
