"""Break the bench's e2e step into host / device parts (c2, pinned host leaves)."""
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

w = bench.workload("c2")
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
for rep in range(6):
    ctx.load_workload(w)
    ctx.schedule(cc.CC_TREE)
    for u, h in host.items():
        ctx.set_leaf(u, h)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(cs)
    t0 = time.perf_counter()
    st = ctx.execute(0)
    t1 = time.perf_counter()
    e1.record(cs)
    ptr, n_corr, ids = ctx.correlator_device_ptr()
    view = bench._device_view(ptr, (n_corr, w.Lt), dev)
    hc = torch.empty((n_corr, w.Lt), dtype=torch.complex128, pin_memory=True)
    with torch.cuda.stream(cs):
        hc.copy_(view, non_blocking=True)
    cs.synchronize()
    t2 = time.perf_counter()
    e2.record(cs)
    e2.synchronize()
    print("execute: host %.2f ms, device (stats) %.2f ms, copies %.2f ms; event e0->e1 %.2f ms, e0->e2 %.2f ms; "
          "after-execute host %.2f ms" % ((t1 - t0) * 1e3, st["seconds"] * 1e3, st["copy_seconds"] * 1e3,
                                        e0.elapsed_time(e1), e0.elapsed_time(e2), (t2 - t1) * 1e3))
os._exit(0)
