"""Run one dataflow replay with a host watchdog that prints the executor's progress."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import dags  # noqa: E402
from oracle import values  # noqa: E402
from oracle.dag import Dag  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = {"c1": dags.config_c1(), "c2s": dags.config_c2(N=40, Lt=3, n_loop4=80, n_loop2=6, n_corr=4)}[name]
dag = Dag(w)
ctx = cc.Context(0, torch.empty(256 << 20, dtype=torch.uint8, device="cuda"))
ctx.load_workload(w)
ctx.schedule(cc.CC_TREE)
keep = []
dev = "--dev" in sys.argv
for u, n in dag.nodes.items():
    if n.child:
        continue
    v = values.synthetic_leaf(w, u, n.op)
    if dev:
        d = torch.from_numpy(v.view(np.float64).ravel().copy()).cuda()
        keep.append(d)
        ctx.set_leaf_device(u, d)
    else:
        h = torch.empty(v.size * 2, dtype=torch.float64, pin_memory=True)
        h.numpy()[:] = v.view(np.float64).ravel()
        keep.append(h)
        ctx.set_leaf(u, h)
print("plan ops:", ctx.plan_ops()[:12], flush=True)
ctx.execute_async(0)
for i in range(8):
    time.sleep(0.5)
    print("state", i, ctx.dataflow_state()[:40], flush=True)
torch.cuda.synchronize()
print("done", flush=True)
os._exit(0)
