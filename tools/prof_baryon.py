"""Stand-alone baryon GEMMs at c4's shape (Lt = 1, N = 128, S = 64: BM1 M = S N^2 = 2^20 rows,
BB2 K = S N^2 = 2^20) on the FP64 DMMA kernel and the tcgen05 Ozaki engine: host-clock times (synchronised; ms-scale launches)
and, under ncu, one launch of each for --set full.  python tools/prof_baryon.py [reps]"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
Lt, N, S = 1, 128, 64
dev = torch.device("cuda:0")
ctx = cc.Context(0, torch.empty(2 << 30, dtype=torch.uint8, device=dev))
nb = Lt * S * N * N * N
A = torch.rand(2 * nb, dtype=torch.float64, device=dev) - 0.5   # baryon [Lt][S][N][N][N]
B = torch.rand(2 * nb, dtype=torch.float64, device=dev) - 0.5
M = torch.rand(2 * Lt * N * N, dtype=torch.float64, device=dev) - 0.5
Cm = torch.empty(2 * Lt * N * N, dtype=torch.float64, device=dev)
Cb = torch.empty(2 * nb, dtype=torch.float64, device=dev)
ws = torch.empty(max(cc.cc_gemm_ozaki_workspace_bytes(op, Lt, N, S, 6) for op in (cc.CC_BM1, cc.CC_BB2)),
                 dtype=torch.uint8, device=dev)
flops = 8.0 * Lt * S * N ** 4
runs = [("BB2 DMMA (zgemm, split-K)", lambda: ctx.bb2(A, B, Cm, Lt, N, S)),
        ("BM1 DMMA (zgemm)", lambda: ctx.bm1(A, M, Cb, Lt, N, S)),
        ("BB2 Ozaki s=6", lambda: ctx.gemm_ozaki(cc.CC_BB2, A, B, Cm, Lt, N, S, 6, ws)),
        ("BM1 Ozaki s=6", lambda: ctx.gemm_ozaki(cc.CC_BM1, A, M, Cb, Lt, N, S, 6, ws))]
for name, f in runs:
    f()
    torch.cuda.synchronize()   # the kernels run on the context's stream: time by host clock
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    print("%-28s %8.3f ms  %6.1f TF/s (8 flop / complex MAC)" % (name, ms, flops / (ms * 1e-3) / 1e12), flush=True)
