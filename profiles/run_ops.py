"""Runner for the ncu captures of the scan-application kernels
(profiles/r01_ops_*_full.txt):
    ncu --set full -k regex:<kernel> -s 1 -c 1 python profiles/run_ops.py <op>
op: split (2^28, fp16 payload + indices), compress (2^28 fp16, no indices), sort (2^24 fp16
keys), sort_rows (512 C4 rows fp32 descending), top_p (1024 C4 rows, p=0.9), shard (C5 shard of 2^29 elements: block sums + row-kernel
pass), rows_short (2^20 x 32 and 2^15 x 4096 fp32 rows), rows_few (8 x 2^24 fp32 rows:
segmented MCScan)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

op = sys.argv[1]
if op == "split":
    n = 1 << 28
    f = torch.empty(n, dtype=torch.int8, device="cuda")
    inputs.fill_device(inputs.I8_FLAG, 2, 0, n, 0, f)
    x = torch.randn(n, device="cuda").half()
    for _ in range(2):
        S.split(x, f)
elif op == "compress":
    n = 1 << 28
    f = torch.empty(n, dtype=torch.int8, device="cuda")
    inputs.fill_device(inputs.I8_FLAG, 2, 0, n, 0, f)
    x = torch.randn(n, device="cuda").half()
    for _ in range(2):
        S.compress(x, f)
elif op == "rows_short":
    for R, C in ((1 << 20, 32), (1 << 15, 4096)):
        X = torch.randn(R, C, device="cuda")
        for _ in range(2):
            S.rows(X)
elif op == "rows_few":
    X = torch.randn(8, 1 << 24, device="cuda")
    for _ in range(2):
        S.rows(X)
elif op == "sort":
    k = torch.randn(1 << 24, device="cuda").half()
    for _ in range(2):
        S.radix_sort(k)
elif op == "sort_rows":  # 512 C4 rows, fp32 descending (the top-p sort path's row sort)
    P = torch.empty((512, 131072), dtype=torch.float32, device="cuda")
    inputs.fill_device(inputs.F32_SOFTMAX, 3, 0, 512, 131072, P)
    for _ in range(2):
        S.radix_sort_rows(P, descending=True)
elif op == "top_p":
    P = torch.empty((1024, 131072), dtype=torch.float32, device="cuda")
    inputs.fill_device(inputs.F32_SOFTMAX, 3, 0, 1024, 131072, P)
    u = torch.rand(1024, device="cuda")
    for _ in range(2):
        S.top_p_sample(P, 0.9, u)
elif op == "shard":
    m = 1 << 29
    x = torch.empty(m, dtype=torch.float32, device="cuda")
    inputs.fill_device(inputs.F32_NORMAL, 4, m, m, 0, x)
    ws = S.shard_workspace(x)
    c = torch.ones(1, dtype=torch.float64, device="cuda")
    for _ in range(2):
        S.shard_reduce(x, ws=ws)
        S.shard_scan(x, carry_in=c, ws=ws)
torch.cuda.synchronize()
