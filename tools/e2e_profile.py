"""Where the end-to-end (pinned host leaves) time goes for a bench workload: schedule, first
execute (plan preparation included), prepared replays, a pure H2D copy of the same bytes,
and the dataflow timeline (when items became ready = when their leaves arrived)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import dags  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = bench.workload(cfg)
dev = torch.device("cuda:0")
streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
arena = torch.empty(6 << 30, dtype=torch.uint8, device=dev)
ctx = cc.Context(0, arena, streams=streams)
host = {}
for n in w.nodes:
    if n[1] in (dags.LEAF_M, dags.LEAF_B):
        shape = bench.leaf_shape(w, n[1])
        per_t = int(np.prod(shape[1:]))
        d = torch.empty(2 * w.Lt * per_t, dtype=torch.float64, device=dev)
        ctx.fill_synthetic(d, w.Lt * per_t, w.data_seed, n[0], 0, w.leaf_mode, bench.leaf_sigma(w, n[1]))
        h = torch.empty(d.numel(), dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize()
        h.copy_(d)
        host[n[0]] = h
torch.cuda.synchronize()
nbytes = sum(h.numel() * 8 for h in host.values())

t0 = time.perf_counter()
ctx.load_workload(w)
order, pst = ctx.schedule(cc.CC_TREE)
t1 = time.perf_counter()
for u, h in host.items():
    ctx.set_leaf(u, h)
st = ctx.execute(0)
t2 = time.perf_counter()
print("load+schedule %.2f ms; first execute %.2f ms wall (%.2f ms device); h2d %.1f MB"
      % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, st["seconds"] * 1e3, st["h2d_bytes"] / 1e6))
for _ in range(3):
    ctx.schedule(cc.CC_TREE)          # invalidates the plan: the next execute prepares again
    t3 = time.perf_counter()
    st = ctx.execute(0)
    t4 = time.perf_counter()
    print("re-prepared execute: %.2f ms wall, %.2f ms device (time to solution), copies done at %.2f ms"
          % ((t4 - t3) * 1e3, st["seconds"] * 1e3, st["copy_seconds"] * 1e3))
for _ in range(3):
    t3 = time.perf_counter()
    st = ctx.execute(0)
    t4 = time.perf_counter()
    print("prepared execute: %.2f ms wall, %.2f ms device, copies done at %.2f ms"
          % ((t4 - t3) * 1e3, st["seconds"] * 1e3, st["copy_seconds"] * 1e3))
# pure H2D of the same bytes on the H2D stream
dst = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(streams[1]):
        e0.record()
        off = 0
        for h in host.values():
            dst[off:off + h.numel()].copy_(h, non_blocking=True)
            off += h.numel()
        e1.record()
    e1.synchronize()
    print("pure H2D of %.1f MB: %.2f ms (%.1f GB/s)" % (nbytes / 1e6, e0.elapsed_time(e1), nbytes / e0.elapsed_time(e1) / 1e6))
ex = ctx.execute(cc.EXEC_PROFILE)
gp, tp = ctx.dataflow_profile()
a = np.vstack([gp, tp]).astype(np.float64)
tb = a[:, 0].min()
rd = np.sort((a[:, 1] - tb) / 1e3)
en = (a[:, 2] - tb) / 1e3
print("profiled execute %.2f ms; item ready-time percentiles (us) 1/10/50/90/99/100: %s; last end %.0f us"
      % (ex["seconds"] * 1e3, np.round(np.percentile(rd, [1, 10, 50, 90, 99, 100]), 0), en.max()))
g = gp.astype(np.float64)
print("gemm first ready %.0f us, gemm ready 50%% at %.0f us, last gemm end %.0f us"
      % ((g[:, 1].min() - tb) / 1e3, (np.median(g[:, 1]) - tb) / 1e3, (g[:, 2].max() - tb) / 1e3))
tpf = tp.astype(np.float64)
print("bin(ms)  gemm_done  trace_done  trace_ready")
span = en.max()
for k in range(int(span // 500) + 1):
    lo, hi = tb + k * 500e3, tb + (k + 1) * 500e3
    print("%5.1f  %8d  %8d  %8d" % (k * 0.5, ((g[:, 2] >= lo) & (g[:, 2] < hi)).sum(),
                                   ((tpf[:, 2] >= lo) & (tpf[:, 2] < hi)).sum(),
                                   ((tpf[:, 1] >= lo) & (tpf[:, 1] < hi)).sum()))
os._exit(0)
