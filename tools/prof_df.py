"""Run the bench workload's dataflow step a few times with device-resident leaves (no copies, so
ncu's kernel serialisation cannot block the worker on a copy flag) — for ncu --set full of
df_worker.  Usage: ncu ... -k regex:df_worker -s 1 -c 1 python tools/prof_df.py [config]"""
import os
import sys

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
arena = torch.empty(int(float(os.environ.get("PROF_ARENA_GB", "6")) * (1 << 30)), dtype=torch.uint8, device=dev)
ctx = cc.Context(0, arena, streams=streams)
ctx.load_workload(w)
ctx.schedule(cc.CC_TREE)
keep = []
for n in w.nodes:
    if n[1] in (dags.LEAF_M, dags.LEAF_B):
        shape = bench.leaf_shape(w, n[1])
        per_t = int(np.prod(shape[1:]))
        d = torch.empty(2 * w.Lt * per_t, dtype=torch.float64, device=dev)
        ctx.fill_synthetic(d, w.Lt * per_t, w.data_seed, n[0], 0, w.leaf_mode, bench.leaf_sigma(w, n[1]))
        ctx.set_leaf_device(n[0], d)
        keep.append(d)
torch.cuda.synchronize()
for _ in range(3):
    st = ctx.execute(0)
print("done", st["seconds"] * 1e3, "ms")
