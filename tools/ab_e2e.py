"""A/B of executor options on the bench's e2e step (c2 from pinned host leaves: load, schedule,
set_leaf, cc_execute with the H2D inside, correlators read back; CUDA events on the compute
stream, median of --reps).  python tools/ab_e2e.py [--reps 8] 'h2d_flag_group=1' 'h2d_flag_group=4' ..."""
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

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--config", default="c2")
ap.add_argument("variants", nargs="+")
a = ap.parse_args()
w = bench.workload(a.config)
dev = torch.device("cuda:0")
streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
cs = streams[0]
ctx = cc.Context(0, torch.empty(6 << 30, dtype=torch.uint8, device=dev), streams=streams)
host = {}
for n in w.nodes:
    if n[1] in (dags.LEAF_M, dags.LEAF_B):
        cnt = int(np.prod(bench.leaf_shape(w, n[1])))
        d = torch.empty(2 * cnt, dtype=torch.float64, device=dev)
        ctx.fill_synthetic(d, cnt, w.data_seed, n[0], 0, w.leaf_mode, bench.leaf_sigma(w, n[1]))
        h = torch.empty(2 * cnt, dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize()
        h.copy_(d)
        host[n[0]] = h
torch.cuda.synchronize()
base = ctx.options()
for v in a.variants:
    opts = dict(base)
    for kv in v.split(","):
        k, x = kv.split("=")
        opts[k] = type(base[k])(float(x))
    ctx.set_options(**opts)
    ts, cd, ref = [], [], None
    for rep in range(a.reps + 1):
        ctx.load_workload(w)
        ctx.schedule(cc.CC_TREE)
        for u, h in host.items():
            ctx.set_leaf(u, h)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        st = ctx.execute(0)
        ptr, n_corr, ids = ctx.correlator_device_ptr()
        view = bench._device_view(ptr, (n_corr, w.Lt), dev)
        hc = torch.empty((n_corr, w.Lt), dtype=torch.complex128, pin_memory=True)
        with torch.cuda.stream(cs):
            hc.copy_(view, non_blocking=True)
        e1.record(cs)
        e1.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
            cd.append(st["copy_seconds"] * 1e3)
        ref = hc.numpy().copy() if ref is None else ref
    print("%-32s e2e median %.3f ms min %.3f ms, copies done %.3f ms" % (v, np.median(ts), np.min(ts), np.median(cd)),
          flush=True)
os._exit(0)
