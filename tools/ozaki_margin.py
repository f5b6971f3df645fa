"""Measured error margin of the Ozaki BB2 at c4's K = S N^2 = 2^20 (N = 128, S = 64) for 4..7
slices, random-phase and phase-limited leaves, against the oracle's BB2 (numpy complex128):
max |gpu - oracle| / (|A| |B| product scale) and the DMMA engine for reference (V-4, V-6)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import rng as srng  # noqa: E402
from oracle import values  # noqa: E402

N, S, Lt = 128, 64, 1
shape = (Lt, S, N, N, N)
ctx = cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
for mode, name in ((srng.MODE_RANDOM_PHASE, "random phase"), (0, "phase-limited")):
    A = np.empty(shape, complex)
    B = np.empty(shape, complex)
    sig = srng.baryon_sigma(N, S)
    srng.leaf_values_into(A, 7, 101, 0, sig, mode)
    srng.leaf_values_into(B, 7, 102, 0, sig, mode)
    want = values.bb2(A, B)
    scale = values.bb2(np.abs(A).astype(complex), np.abs(B).astype(complex)).real
    dA = torch.from_numpy(A.view(np.float64).ravel().copy()).cuda()
    dB = torch.from_numpy(B.view(np.float64).ravel().copy()).cuda()
    C = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
    rows = []
    for s in (0, 4, 5, 6, 7):
        if s == 0:
            ctx.bb2(dA, dB, C, Lt, N, S)
        else:
            ws = torch.empty(cc.cc_gemm_ozaki_workspace_bytes(cc.CC_BB2, Lt, N, S, s), dtype=torch.uint8, device="cuda")
            ctx.gemm_ozaki(cc.CC_BB2, dA, dB, C, Lt, N, S, s, ws)
        torch.cuda.synchronize()
        got = C.cpu().numpy().view(np.complex128).reshape(Lt, N, N)
        e = np.abs(got - want)
        print("%-14s %-10s max err / |A||B| scale %.2e, max err / |C| %.2e" % (
            name, "DMMA" if s == 0 else "Ozaki s=%d" % s, float((e / scale).max()),
            float((e / np.maximum(np.abs(want), 1e-300)).max())), flush=True)
os._exit(0)
