"""Per-item phase times of trace items in a profiled dataflow replay of the bench workload:
claim -> ready (deps), ready -> first stage consumed, stage loop, loop end -> published; in
the GEMM phase and in the trace tail."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import dags, rng as srng  # noqa: E402

w = dags.config_c2()
dev = torch.device("cuda:0")
ctx = cc.Context(0, torch.empty(6 << 30, dtype=torch.uint8, device=dev))
ctx.load_workload(w)
ctx.schedule(cc.CC_TREE)
keep = []
for (u, op, a, b, s) in w.nodes:
    if op not in (dags.LEAF_M, dags.LEAF_B):
        continue
    n = w.Lt * w.N * w.N
    d = torch.empty(2 * n, dtype=torch.float64, device=dev)
    ctx.fill_synthetic(d, n, w.data_seed, u, 0, 0, srng.meson_sigma(w.N))
    keep.append(d)
    ctx.set_leaf_device(u, d)
for _ in range(3):
    ctx.execute(0)
ctx.execute(cc.EXEC_PROFILE)
gp, tp = ctx.dataflow_profile()
g = gp.astype(np.float64)
t = tp.astype(np.float64)
t0 = min(g[:, 0].min(), t[:, 0].min())
g_end = g[:, 2].max()
print("GEMM items end at %.1f us, trace items end at %.1f us" % ((g_end - t0) / 1e3, (t[:, 2].max() - t0) / 1e3))
for name, m in (("during GEMMs", t[:, 2] < g_end), ("tail", t[:, 2] >= g_end)):
    a = t[m]
    if not len(a):
        continue
    ph = [(a[:, 1] - a[:, 0]), (a[:, 4] - a[:, 1]), (a[:, 5] - a[:, 4]), (a[:, 2] - a[:, 5])]
    print("%-13s %6d items: claim->ready %.2f us, ready->first data %.2f us, 16-stage loop %.2f us, loop end->published %.2f us"
          % ((name, len(a)) + tuple(np.median(x) / 1e3 for x in ph)))
    # concurrency: trace items in flight per SM
    sm = a[:, 3]
    print("              items per SM %.1f, SMs %d" % (len(a) / len(np.unique(sm)), len(np.unique(sm))))
os._exit(0)
