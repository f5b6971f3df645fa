"""Stand-alone timing: MM1 on FP64 DMMA (cc_mm1) vs Ozaki-split INT8 tcgen05 (cc_mm1_ozaki),
and the raw INT8 tcgen05 GEMM.  CUDA events on the ctx compute stream, L2 flushed before each
timed launch, median of reps.  Algorithmic flops: 8 Lt N^3 per MM1 (8 per complex MAC)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402


def timeit(fn, stream, flush, reps=10):
    ts = []
    for _ in range(reps + 2):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream(device=dev)
    arena = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    ctx = cc.Context(0, arena, streams=[s, torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = []
    for (Lt, N) in ((64, 128), (16, 256), (8, 512), (2, 1024)):
        A = torch.rand(Lt * N * N * 2, dtype=torch.float64, device=dev) + 0.5
        B = torch.rand(Lt * N * N * 2, dtype=torch.float64, device=dev) + 0.5
        C = torch.empty_like(A)
        fl = 8.0 * Lt * N ** 3
        row = {"Lt": Lt, "N": N}
        with torch.cuda.stream(s):
            t = timeit(lambda: ctx.mm1(A, B, C, Lt, N), s, flush)
            row["dmma_us"] = t * 1e6
            row["dmma_tflops"] = fl / t / 1e12
            for ns in (5,):
                ws = torch.empty(cc.cc_mm1_ozaki_workspace_bytes(Lt, N, ns), dtype=torch.uint8, device=dev)
                t = timeit(lambda: ctx.mm1_ozaki(A, B, C, Lt, N, ns, ws), s, flush)
                row["ozaki%d_us" % ns] = t * 1e6
                row["ozaki%d_tflops_equiv" % ns] = fl / t / 1e12
        print(json.dumps(row), flush=True)
        out.append(row)
    for (M, Nn, K) in ((8192, 8064, 8192), (16384, 8064, 4096)):
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
        b = torch.randint(-127, 128, (Nn, K), dtype=torch.int8, device=dev)
        c = torch.empty((M, Nn), dtype=torch.int32, device=dev)
        with torch.cuda.stream(s):
            t = timeit(lambda: ctx.i8gemm_tn(a, b, c, M, Nn, K), s, flush, reps=5)
        row = {"i8gemm": [M, Nn, K], "us": t * 1e6, "tops": 2.0 * M * Nn * K / t / 1e12}
        print(json.dumps(row), flush=True)
        out.append(row)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "ozaki_bench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
