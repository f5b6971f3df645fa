"""Timeline summary of one dataflow replay of the bench workload (flags bit 5)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import dags, rng as srng  # noqa: E402

import bench  # noqa: E402
w = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
dev = torch.device("cuda:0")
ctx = cc.Context(0, torch.empty(int(float(os.environ.get("PROF_ARENA_GB", "6")) * (1 << 30)), dtype=torch.uint8, device=dev))
ctx.load_workload(w)
ctx.schedule(cc.CC_TREE)
keep = []
for (u, op, a, b, s) in w.nodes:
    if op not in (dags.LEAF_M, dags.LEAF_B):
        continue
    n = w.Lt * w.N * w.N * (1 if op == dags.LEAF_M else w.S * w.N)
    d = torch.empty(2 * n, dtype=torch.float64, device=dev)
    sig = srng.meson_sigma(w.N) if op == dags.LEAF_M else srng.baryon_sigma(w.N, w.S)
    ctx.fill_synthetic(d, n, w.data_seed, u, 0, 0, sig)
    keep.append(d)
    ctx.set_leaf_device(u, d)
ts = []
for _ in range(5):
    ts.append(ctx.execute(0)["seconds"] * 1e3)
print("plain executes (ms):", np.round(ts, 3))
ex = ctx.execute(cc.EXEC_PROFILE)
gp, tp, psm = ctx.dataflow_profile(per_sm=True)
tot = psm[:, :4].sum(axis=1).astype(np.float64)
print("GEMM epilogue (thread 0, included in work G): %.0f cycles per item, %.1f%% of consumer time"
      % (psm[:, 7].sum() / max(psm[:, 4].sum() / 8, 1), 100 * psm[:, 7].sum() / tot.sum()))
print("consumer warps (thread 0, clock64): stage wait %.1f%%, stage math %.1f%%; %d GEMM stages: %.0f wait + %.0f "
      "math cycles each; trace stages per trace warp (4 per CTA): %s"
      % (100 * psm[:, 0].sum() / tot.sum(), 100 * psm[:, 2].sum() / tot.sum(), psm[:, 4].sum(),
         psm[:, 0].sum() / max(psm[:, 4].sum(), 1), psm[:, 2].sum() / max(psm[:, 4].sum(), 1),
         psm[:, 8:12].sum(axis=0).tolist()))
if psm.shape[1] > 13 and psm[:, 13].sum() > 0:
    ntr = psm[:, 8].sum()
    print("trace warp 0 (clock64): waiting for stage data %.0f cycles per stage, computing %.0f cycles per stage "
          "(%d stages)" % (psm[:, 12].sum() / max(ntr, 1), psm[:, 13].sum() / max(ntr, 1), ntr))
g0 = np.vstack([gp, tp])
g, t = g0[g0[:, 6] == 0], g0[g0[:, 6] == 1]
t0 = min(g[:, 0].min() if len(g) else 2**63, t[:, 0].min() if len(t) else 2**63)
t1 = max(g[:, 2].max() if len(g) else 0, t[:, 2].max() if len(t) else 0)
span = (t1 - t0) / 1e3
print("execute %.3f ms, worker span %.3f ms" % (ex["seconds"] * 1e3, span / 1e3))
for name, a in (("gemm", g), ("trace", t)):
    if not len(a):
        continue
    a = a.astype(np.float64)
    wait = (a[:, 1] - a[:, 0]) / 1e3
    work = (a[:, 2] - a[:, 4]) / 1e3
    sms = len(np.unique(a[:, 3]))
    print("%-5s items %6d on %3d SMs: work %.1f us avg (sum %.2f ms), dep-wait %.2f us avg (sum %.2f ms), "
          "busy %.1f%% of %d SMs x span" % (name, len(a), sms, work.mean(), work.sum() / 1e3, wait.mean(),
                                              wait.sum() / 1e3, 100 * work.sum() / (sms * span), sms))
    # per-SM timeline occupancy gaps
    q = np.percentile(work, [10, 50, 90, 99])
    print("      work percentiles 10/50/90/99: %s us" % np.round(q, 1))
    # consumer side: start (info received) -> first data -> end of stage loop -> end
    wait_data = (a[:, 7] - a[:, 4]) / 1e3
    loop = (a[:, 5] - a[:, 7]) / 1e3
    epi = (a[:, 2] - a[:, 5]) / 1e3
    busy = (a[:, 2] - a[:, 4]) / 1e3
    print("      consumer: wait first data %.2f us, stage loop %.2f us, epilogue+publish %.2f us, total %.2f us"
          % (wait_data.mean(), loop.mean(), epi.mean(), busy.mean()))
    print("      consumer busy %.1f%% of SM x span" % (100 * busy.sum() / (sms * span)))
    print("      wait-first-data percentiles 10/50/90/99: %s us" % np.round(np.percentile(wait_data, [10, 50, 90, 99]), 2))
    first = (a[:, 0].min() - t0) / 1e3
    last = (a[:, 2].max() - t0) / 1e3
    print("      first dispatch at %.1f us, last end at %.1f us" % (first, last))
# per SM: consumer timeline (all kinds): loop time vs gaps between one item's loop end and the
# next item's first data
allp = g0.astype(np.float64)
loop_sum, gap_sum = 0.0, 0.0
for smv in np.unique(allp[:, 3]):
    r = allp[allp[:, 3] == smv]
    r = r[np.argsort(r[:, 4])]
    loop_sum += (r[:, 5] - r[:, 7]).sum()
    gap_sum += (r[1:, 7] - r[:-1, 5]).sum()
print("consumers: stage loops %.1f%%, between loops %.1f%% of summed per-SM time"
      % (100 * loop_sum / (loop_sum + gap_sum), 100 * gap_sum / (loop_sum + gap_sum)))
# time bins: items running and mean duration per 0.5 ms
span_ns = t1 - t0
binw = max(500000, int(span_ns // 40))   # at most ~40 bins
nb = int(span_ns // binw) + 1
print("bin(ms)  gemm_items  gemm_us  trace_items  trace_us  trace_SMs")
for k in range(nb):
    lo, hi = t0 + k * binw, t0 + (k + 1) * binw
    row = []
    for a in (g, t):
        m = (a[:, 1] >= lo) & (a[:, 1] < hi)
        d = (a[m, 2].astype(np.float64) - a[m, 1]) / 1e3
        row.append((int(m.sum()), d.mean() if m.any() else 0.0, len(np.unique(a[m, 3]))))
    print("%5.1f  %8d  %7.1f  %8d  %7.1f  %4d" % (k * binw / 1e6, row[0][0], row[0][1], row[1][0], row[1][1], row[1][2]))
os._exit(0)
