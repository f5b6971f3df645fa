"""One rank of the multi-process peer-tier check (tests/test_gpu_multirank.py), launched by
torch.distributed.run with N ranks on the GPUs there are (several ranks may share one GPU:
CUDA IPC maps a buffer of another process on the same device the same way as a peer GPU's).

Each rank runs its TREES part of a small c4 DAG under a capacity that forces evictions, with
the peer-HBM tier (E-10: it evicts into the next rank's lent HBM) and cross-GPU leaf sharing
(E-11: every leaf is loaded over PCIe once, by its owner rank, and read from the owner's HBM by
the others).  Rank 0 sums the parts' correlators and checks them against the oracle; every rank
checks that its executor moved exactly its plan's bytes on each path.  Prints one JSON line.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from synth import dags, rng as srng  # noqa: E402
from paper_2511_02257_b200 import cc  # noqa: E402
from paper_2511_02257_b200.dist import setup_peer_tier, SharedLeaves, close_buffers  # noqa: E402


def main():
    flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    mode = sys.argv[2] if len(sys.argv) > 2 else "both"      # plain | tier | leaves | both
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    w = dags.config_c4(N=16, Lt=2, S=4, n_snk=3, n_src=3, n_mes=4, n_trees=24)
    baryon = 16 * w.Lt * w.S * w.N ** 3
    cap, peer_cap = 5 * baryon, 2 * baryon
    arena = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    ctx = cc.Context(dev.index, arena)
    ctx.load_workload(w)
    ctx.partition(world, rank, cc.PART_TREES)
    host = {}
    for n in w.nodes:
        if n[1] in (dags.LEAF_M, dags.LEAF_B):
            shape = (w.Lt, w.N, w.N) if n[1] == dags.LEAF_M else (w.Lt, w.S, w.N, w.N, w.N)
            cnt = int(np.prod(shape))
            d = torch.empty(2 * cnt, dtype=torch.float64, device=dev)
            sigma = srng.meson_sigma(w.N) if n[1] == dags.LEAF_M else srng.baryon_sigma(w.N, w.S)
            ctx.fill_synthetic(d, cnt, w.data_seed, n[0], 0, w.leaf_mode, sigma)
            torch.cuda.synchronize(dev)      # the generator runs on the library's stream
            host[n[0]] = d.cpu().pin_memory()
    tier_ptrs, peer_leaves = [], []
    if mode in ("tier", "both"):
        lent, tier_ptrs = setup_peer_tier(ctx, 8 << 20, dev)
    else:
        peer_cap = 0
    shared = None
    if mode in ("leaves", "both"):
        sizes = {u: h.numel() * h.element_size() for u, h in host.items()}
        shared = SharedLeaves(ctx, sizes, host, dev)
        shared.stage()
        peer_leaves = shared.ids
    else:
        for u, h in host.items():
            ctx.set_leaf(u, h)
    _, st = ctx.schedule(cc.CC_TREE, cap_bytes=cap, peer_cap_bytes=peer_cap, peer_leaves=peer_leaves)
    ex = ctx.execute(flags)
    ok_bytes = (ex["h2d_bytes"], ex["d2h_bytes"], ex["p2p_in_bytes"], ex["p2p_out_bytes"]) == \
        (st["h2d_bytes"], st["d2h_bytes"], st["p2p_in_bytes"], st["p2p_out_bytes"])
    _, n_corr, ids = ctx.correlator_device_ptr()
    part = {int(c): ctx.correlator(c, w.Lt) for c in ids}
    allp = [None] * world
    dist.all_gather_object(allp, (part, ok_bytes, st["evictions"], st["p2p_out_count"], st["h2d_bytes"]))
    dist.barrier()                          # every rank's executes are done before unmapping
    if tier_ptrs:
        close_buffers(tier_ptrs)
    if shared is not None:
        shared.close()
    if rank == 0:
        total = {}
        for p, *_ in allp:
            for c, v in p.items():
                total[c] = total.get(c, 0) + v
        print(json.dumps({"world": world, "corr": {str(c): [list(map(float, v.real)), list(map(float, v.imag))]
                                                   for c, v in total.items()},
                          "bytes_ok": all(a[1] for a in allp), "evictions": [a[2] for a in allp],
                          "p2p_out": [a[3] for a in allp], "h2d_bytes": [a[4] for a in allp]}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
