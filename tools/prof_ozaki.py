"""One Ozaki MM1 per size for ncu (split kernels + tcgen05 GEMM)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402

sizes = [(int(a), int(b)) for a, b in (x.split("x") for x in (sys.argv[1:] or ["2x1024", "64x128"]))]
dev = torch.device("cuda:0")
ctx = cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device=dev))
for Lt, N in sizes:
    A = torch.rand(Lt * N * N * 2, dtype=torch.float64, device=dev) + 0.5
    B = torch.rand(Lt * N * N * 2, dtype=torch.float64, device=dev) + 0.5
    C = torch.empty_like(A)
    ws = torch.empty(cc.cc_mm1_ozaki_workspace_bytes(Lt, N, 5), dtype=torch.uint8, device=dev)
    for _ in range(2):
        ctx.mm1_ozaki(A, B, C, Lt, N, 5, ws)
    torch.cuda.synchronize()
