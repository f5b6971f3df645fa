"""A/B of executor options on the bench workload (device-resident leaves, graph replay, L2
flushed before every replay; CUDA events on the compute stream).
python tools/ab_options.py [--config c2] [--reps 20] 'slice_major=0' 'slice_major=1' ..."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import dags  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--flags", type=int, default=1)
    ap.add_argument("--arena-gb", type=float, default=6)
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    w = bench.workload(a.config)
    dev = torch.device("cuda:0")
    streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
    arena = torch.empty(int(a.arena_gb * (1 << 30)), dtype=torch.uint8, device=dev)
    ctx = cc.Context(0, arena, streams=streams)
    ctx.load_workload(w)
    ctx.schedule(cc.CC_TREE)
    keep = []
    for n in w.nodes:
        if n[1] in (dags.LEAF_M, dags.LEAF_B):
            per_t = int(np.prod(bench.leaf_shape(w, n[1])[1:]))
            d = torch.empty(2 * w.Lt * per_t, dtype=torch.float64, device=dev)
            ctx.fill_synthetic(d, w.Lt * per_t, w.data_seed, n[0], 0, w.leaf_mode, bench.leaf_sigma(w, n[1]))
            ctx.set_leaf_device(n[0], d)
            keep.append(d)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cs = streams[0]
    ref = None
    base = ctx.options()
    for v in a.variants:
        opts = dict(base)
        for kv in v.split(","):
            k, x = kv.split("=")
            opts[k] = type(base[k])(float(x)) if isinstance(base[k], int) else float(x)
        ctx.set_options(**opts)
        ctx.execute(a.flags)
        ts = []
        for _ in range(a.reps):
            with torch.cuda.stream(cs):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            ctx.execute_async(a.flags)
            e1.record(cs)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        _, n_corr, ids = ctx.correlator_device_ptr()
        vals = np.concatenate([ctx.correlator(c, w.Lt) for c in ids])
        dif = 0.0 if ref is None else float(np.max(np.abs(vals - ref) / np.maximum(np.abs(ref), 1e-300)))
        ref = vals if ref is None else ref
        print("%-40s median %.3f ms  min %.3f ms  (max rel diff vs first %.1e)" % (v, np.median(ts), np.min(ts), dif),
              flush=True)


if __name__ == "__main__":
    main()
