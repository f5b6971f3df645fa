"""Launch the bench's kernels at the bench's shapes a few times (for ncu --set full)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02257_b200 import cc  # noqa: E402

Lt, N = int(os.environ.get("LT", 64)), int(os.environ.get("NN", 128))
dev = torch.device("cuda:0")
ctx = cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device=dev))
A = torch.rand(2 * Lt * N * N, dtype=torch.float64, device=dev)
B = torch.rand(2 * Lt * N * N, dtype=torch.float64, device=dev)
C = torch.empty_like(A)
c = torch.empty(2 * Lt, dtype=torch.float64, device=dev)
for _ in range(4):
    ctx.mm1(A, B, C, Lt, N)
    ctx.tr_mm(A, B, c, Lt, N)
torch.cuda.synchronize()
print("done")
