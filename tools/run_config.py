"""Run a BASELINE config end to end at full size from pinned host leaves: time to solution,
transfers vs the plan, PCIe / FP64 bounds.  (Values: tests/test_gpu_parity.py.)

Usage: python tools/run_config.py c3|c4|c5 [--cap BYTES] [--N N] [--parts P --part p] [--device-leaves]
c5 at N=512/1024 runs one rank's TIME part of the 8-GPU partition (--parts 8) with device-resident
leaves (the full pinned host set would be 32 / 128 GiB).
"""
import argparse
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--cap", type=float, default=None)
    ap.add_argument("--arena-gb", type=float, default=150)
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--parts", type=int, default=1)
    ap.add_argument("--part", type=int, default=0)
    ap.add_argument("--device-leaves", action="store_true")
    ap.add_argument("--ozaki", action="store_true", help="MM1 on the tcgen05 INT8 Ozaki engine (execute flags bit 6)")
    ap.add_argument("--next-use", action="store_true", help="next-use (Belady) eviction, reading E-9")
    ap.add_argument("--op-by-op", action="store_true", help="op-by-op executor (execute flags bit 4)")
    ap.add_argument("--breakdown", action="store_true",
                    help="one more op-by-op execute with every kernel timed (flags bit 1): time per op kind")
    a = ap.parse_args()
    w = {"c3": dags.config_c3, "c4": dags.config_c4, "c5": lambda: dags.config_c5(N=a.N)}[a.config]()
    cap = int(a.cap) if a.cap is not None else (32 * 10 ** 9 if a.config == "c4" else 0)
    dev = torch.device("cuda:0")
    streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
    arena = torch.empty(int(a.arena_gb * (1 << 30)), dtype=torch.uint8, device=dev)
    ctx = cc.Context(0, arena, streams=streams)
    t0 = time.perf_counter()
    ctx.load_workload(w)
    if a.parts > 1:
        ctx.partition(a.parts, a.part, cc.PART_TIME)
    pt0, pt1 = ctx.part_time_range()
    order, st = ctx.schedule(cc.CC_TREE, cap_bytes=cap, evict_next_use=a.next_use)
    t1 = time.perf_counter()
    print("%s%s: %d contractions, plan peak %.2f GB transient %.2f GB, evictions %d, H2D %.2f GB D2H %.2f GB, "
          "schedule+plan %.1f ms" % (w.name, " (next-use eviction)" if a.next_use else "", st["n_contr"], st["peak"] / 1e9, st["transient_peak"] / 1e9,
                                     st["evictions"], st["h2d_bytes"] / 1e9, st["d2h_bytes"] / 1e9,
                                     (t1 - t0) * 1e3), flush=True)
    host = {}
    tmp = None
    for n in w.nodes:
        if n[1] not in (dags.LEAF_M, dags.LEAF_B):
            continue
        shape = bench.leaf_shape(w, n[1])
        if a.device_leaves:
            per_t = int(np.prod(shape[1:]))
            d = torch.empty(2 * (pt1 - pt0) * per_t, dtype=torch.float64, device=dev)
            ctx.fill_synthetic(d, (pt1 - pt0) * per_t, w.data_seed, n[0], pt0 * per_t, w.leaf_mode,
                               bench.leaf_sigma(w, n[1]))
            host[n[0]] = d
            continue
        cnt = int(np.prod(shape))
        if tmp is None or tmp.numel() < 2 * cnt:
            tmp = torch.empty(2 * cnt, dtype=torch.float64, device=dev)
        d = tmp[:2 * cnt]
        ctx.fill_synthetic(d, cnt, w.data_seed, n[0], 0, w.leaf_mode, bench.leaf_sigma(w, n[1]))
        h = torch.empty(2 * cnt, dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize()
        h.copy_(d)
        host[n[0]] = h
    del tmp
    torch.cuda.synchronize()
    for u, h in host.items():
        if a.device_leaves:
            ctx.set_leaf_device(u, h)
        else:
            ctx.set_leaf(u, h)
    print("part %d/%d: time slices [%d, %d), %d trees" % (a.part, a.parts, pt0, pt1, len(ctx.part_trees())), flush=True)
    for rep in range(2):
        ex = ctx.execute((cc.EXEC_OZAKI_MM1 if a.ozaki else 0) | (cc.EXEC_OP_BY_OP if a.op_by_op else 0))
        moved = ex["h2d_bytes"] + ex["d2h_bytes"]
        print("execute %d%s: %.1f ms (copies done %.1f ms); moved %.2f GB -> PCIe bound %.1f ms; flops %.3g -> "
              "FP64 bound %.1f ms" % (rep, " (Ozaki MM1, op-by-op)" if a.ozaki else "", ex["seconds"] * 1e3, ex["copy_seconds"] * 1e3, moved / 1e9,
                                      moved / 55.6e9 * 1e3, ex["flops"], ex["flops"] / 37.0e12 * 1e3), flush=True)
    if a.breakdown:
        ctx.execute(cc.EXEC_TIME_KERNELS | (cc.EXEC_OZAKI_MM1 if a.ozaki else 0))
        secs, cnts = ctx.kernel_times()
        Lt_p, N = pt1 - pt0, w.N
        names = {2: "MM1", 3: "BM1", 4: "BB2", 5: "TR_MM"}
        for k, nm in names.items():
            if cnts[k]:
                extra = ""
                if k == 2:
                    extra = ", %.1f TF/s (8 flop/cMAC)" % (8.0 * Lt_p * N ** 3 * cnts[k] / secs[k] / 1e12)
                if k == 5:   # batched trace launches: count the TR_MM ops of the plan, not the launches
                    n_tr = sum(1 for nd in w.nodes if nd[1] == dags.TR_MM)
                    extra = ", %d traces, %.0f GB/s algorithmic" % (n_tr, 32.0 * Lt_p * N * N * n_tr / secs[k] / 1e9)
                print("  %s: %d launches, %.1f ms%s" % (nm, cnts[k], secs[k] * 1e3, extra), flush=True)
    # values are checked against the oracle by tests/test_gpu_parity.py (tools do not run it)
    os._exit(0)


if __name__ == "__main__":
    main()
