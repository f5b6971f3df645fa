"""c4 (or c5) from pinned host leaves through the dataflow worker with the per-item timeline
(flags bit 5): GEMM- and trace-item busy fractions of the SMs per 50 ms bin, to see where the
worker waits on copies or on traces.
python tools/c4_timeline.py [--cap BYTES] [--lru] [--config c5 --N 256 --cap 0]"""
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
ap.add_argument("--cap", type=float, default=32e9)
ap.add_argument("--lru", action="store_true")
ap.add_argument("--config", default="c4")
ap.add_argument("--N", type=int, default=256)
ap.add_argument("--opt", action="append", default=[], help="executor option k=v (cc_set_options)")
a = ap.parse_args()
w = dags.config_c4() if a.config == "c4" else dags.config_c5(N=a.N)
dev = torch.device("cuda:0")
streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
ctx = cc.Context(0, torch.empty((60 if a.config == "c4" else 150) << 30, dtype=torch.uint8, device=dev), streams=streams)
if a.opt:
    o = ctx.options()
    o.update({k: type(o[k])(float(v)) for k, v in (x.split("=") for x in a.opt)})
    ctx.set_options(**o)
ctx.load_workload(w)
_, st = ctx.schedule(cc.CC_TREE, cap_bytes=int(a.cap), evict_next_use=not a.lru)
host, tmp = {}, None
for n in w.nodes:
    if n[1] not in (dags.LEAF_M, dags.LEAF_B):
        continue
    cnt = int(np.prod(bench.leaf_shape(w, n[1])))
    if tmp is None or tmp.numel() < 2 * cnt:
        tmp = torch.empty(2 * cnt, dtype=torch.float64, device=dev)
    d = tmp[:2 * cnt]
    ctx.fill_synthetic(d, cnt, w.data_seed, n[0], 0, w.leaf_mode, bench.leaf_sigma(w, n[1]))
    h = torch.empty(2 * cnt, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    h.copy_(d)
    host[n[0]] = h
    ctx.set_leaf(n[0], h)
del tmp
ex = ctx.execute(0)
print("plain execute %.1f ms, copies done %.1f ms; plan: evictions %d, H2D %.1f GB" % (
    ex["seconds"] * 1e3, ex["copy_seconds"] * 1e3, st["evictions"], st["h2d_bytes"] / 1e9))
ex = ctx.execute(cc.EXEC_PROFILE)
gp, tp = ctx.dataflow_profile()
g = gp.astype(np.float64)
tr = tp.astype(np.float64)
t0 = min(g[:, 0].min(), tr[:, 0].min() if len(tr) else g[:, 0].min())
end = max(g[:, 2].max(), tr[:, 2].max() if len(tr) else 0)
binw = 50e6
nb = int((end - t0) // binw) + 1


def occupancy(a):
    busy = np.zeros(nb)
    for (s0, e0) in zip(a[:, 4] - t0, a[:, 2] - t0):   # first data -> published
        b0, b1 = int(s0 // binw), int(e0 // binw)
        for b in range(b0, b1 + 1):
            lo, hi = max(s0, b * binw), min(e0, (b + 1) * binw)
            if hi > lo:
                busy[b] += hi - lo
    return busy


bg, bt = occupancy(g), occupancy(tr) if len(tr) else np.zeros(nb)
print("profiled execute %.1f ms; GEMM items %d, trace items %d" % (ex["seconds"] * 1e3, len(g), len(tr)))
print("bin(ms)  GEMM-busy%  trace-busy%  (items first data -> published, of 148 SMs)")
for b in range(nb):
    print("%6.0f  %6.1f  %6.1f" % (b * binw / 1e6, 100 * bg[b] / (148 * binw), 100 * bt[b] / (148 * binw)))
os._exit(0)
