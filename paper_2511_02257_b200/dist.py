"""Multi-GPU plumbing: the one collective of the path.

Each rank executes one part of the DAG (cc_partition: TIME slices or TREES chunks) and
holds its correlator partial [n_corr, Lt_part] (complex128, device buffer of libcc exposed
by cc_correlator_device_ptr).  The only exchange is a sum over ranks: a TIME part writes its
slices into a zero-padded [n_corr, Lt] buffer, a TREES part already covers every slice, and
one all_reduce (NCCL over NVLink on GPUs, gloo in the CPU tests) produces the correlators.
"""
import torch
import torch.distributed as dist


def allreduce_correlators(part, t0, t1, Lt, group=None, out=None):
    """Sum the per-rank correlator partials.  part: complex128 [n_corr, t1 - t0]."""
    if out is None:
        out = torch.zeros((part.shape[0], Lt), dtype=torch.complex128, device=part.device)
    else:
        out.zero_()
    out[:, t0:t1].copy_(part)
    dist.all_reduce(torch.view_as_real(out), group=group)
    return out
