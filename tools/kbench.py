"""Per-kernel timing of the contraction kernels (CUDA events on the launching stream).

python tools/kbench.py [--quick]
Prints TFLOP/s (FP64, 8 real flops per complex MAC) and GB/s against MEASURED peaks.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402


def timeit(fn, stream, reps=10, warm=3, flush=None, inner=20):
    """Median over `reps` of (time of `inner` back-to-back launches)/inner; the stream is kept
    backlogged (a flush kernel queued first) so host launch overhead is not measured."""
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(inner):
            fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / inner)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default=None, help="run only cases of this kind (MM1, BM1, BB2, TR)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    streams = [torch.cuda.Stream() for _ in range(3)]
    arena = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    ctx = cc.Context(0, arena, streams=streams)
    s = streams[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rows = []

    def rnd(n):
        return torch.rand(2 * n, dtype=torch.float64, device=dev)

    cases = [("MM1", 64, 128, 1), ("MM1", 128, 256, 1), ("MM1", 128, 512, 1)]
    if not a.quick:
        cases += [("MM1", 4, 32, 1), ("MM1", 128, 1024, 1), ("BM1", 32, 64, 64), ("BB2", 32, 64, 64),
                  ("BM1", 1, 128, 64), ("BB2", 1, 128, 64), ("TR", 64, 128, 1), ("TR", 128, 1024, 1), ("TR", 8, 1024, 1), ("TR", 16, 512, 1)]
    if a.only:
        cases = [c for c in cases if c[0] == a.only]
    for kind, Lt, N, S in cases:
        if kind == "MM1":
            A, B, C = rnd(Lt * N * N), rnd(Lt * N * N), rnd(Lt * N * N)
            fn = lambda: ctx.mm1(A, B, C, Lt, N)  # noqa: E731
            flops = 8.0 * Lt * N ** 3
            byts = 48.0 * Lt * N * N
        elif kind == "BM1":
            A, B, C = rnd(Lt * S * N ** 3), rnd(Lt * N * N), rnd(Lt * S * N ** 3)
            fn = lambda: ctx.bm1(A, B, C, Lt, N, S)  # noqa: E731
            flops = 8.0 * Lt * S * N ** 4
            byts = 16.0 * Lt * (2 * S * N ** 3 + N * N)
        elif kind == "BB2":
            A, B, C = rnd(Lt * S * N ** 3), rnd(Lt * S * N ** 3), rnd(Lt * N * N)
            fn = lambda: ctx.bb2(A, B, C, Lt, N, S)  # noqa: E731
            flops = 8.0 * Lt * S * N ** 4
            byts = 16.0 * Lt * (2 * S * N ** 3 + N * N)
        else:
            A, B, C = rnd(Lt * N * N), rnd(Lt * N * N), rnd(Lt)
            fn = lambda: ctx.tr_mm(A, B, C, Lt, N)  # noqa: E731
            flops = 8.0 * Lt * N * N
            byts = 32.0 * Lt * N * N
        t = timeit(fn, s, flush=flush, inner=3 if flops > 1e11 else 20)
        r = dict(kind=kind, Lt=Lt, N=N, S=S, us=t * 1e6, tflops=flops / t / 1e12, gbs=byts / t / 1e9)
        rows.append(r)
        print("%-4s Lt=%4d N=%5d S=%3d  %10.1f us  %7.2f TFLOP/s  %8.1f GB/s" %
              (kind, Lt, N, S, r["us"], r["tflops"], r["gbs"]), flush=True)
        del A, B, C
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "kbench.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
