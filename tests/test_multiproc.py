"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path: the C++ partition of
each rank (host-only libcc context) + the correlator all-reduce helper must reproduce the
full correlators.  The oracle stands in for the GPU values of each part (the GPU parity of a
part is tested in test_gpu_parity.py::test_partitions_sum_to_whole)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import dags
from oracle import values, partition
from oracle.dag import Dag

cc = pytest.importorskip("paper_2511_02257_b200.cc")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_02257_b200.dist import allreduce_correlators
        w = dags.config_c2(N=6, Lt=6, n_loop4=40, n_loop2=4, n_corr=3)
        ctx = cc.Context(-1)
        ctx.load_workload(w)
        ctx.partition(world, rank, mode)
        trees = ctx.part_trees()
        order, st = ctx.schedule(cc.CC_TREE)
        full = Dag(w)
        corr_ids = sorted({c for (c, _, _, _) in w.terms})
        if mode == cc.PART_TIME:
            t0, t1 = partition.time_range(w.Lt, world, rank)
            r, c = values.run_workload(w, full, t_range=(t0, t1))
        else:
            t0, t1 = 0, w.Lt
            sub = partition.sub_workload(w, trees)
            r, c = values.run_workload(sub, Dag(sub))
        part = torch.zeros((len(corr_ids), t1 - t0), dtype=torch.complex128)
        for k, cid in enumerate(corr_ids):
            if cid in c:
                part[k] = torch.from_numpy(np.asarray(c[cid]))
        tot = allreduce_correlators(part, t0, t1, w.Lt)
        if rank == 0:
            _, want = values.run_workload(w, full)
            ok = all(np.allclose(tot[k].numpy(), want[cid], rtol=1e-12, atol=1e-14) for k, cid in enumerate(corr_ids))
            result_q.put((ok, len(trees)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
def test_two_rank_partition_allreduce(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ok, n = q.get(timeout=10)
    assert ok and n > 0
