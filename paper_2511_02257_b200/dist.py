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


# ---- peer-HBM tier and cross-GPU leaf sharing (readings E-10, E-11) -------
# Rank processes exchange CUDA IPC handles of device buffers (cc_ipc_export / cc_ipc_open) over
# the process group; the copies themselves are issued by the library's executors.

def exchange_buffers(buf, group=None):
    """Every rank's `buf` as an address in this process: entry r = rank r's buffer (own: local
    address; others: an IPC mapping, to be released with close_buffers)."""
    from . import cc
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    h, off = cc.ipc_export(buf)
    allh = [None] * world
    dist.all_gather_object(allh, (h, off), group=group)
    return [buf.data_ptr() if r == rank else cc.ipc_open(hh, oo) for r, (hh, oo) in enumerate(allh)]


def close_buffers(ptrs, group=None):
    from . import cc
    rank = dist.get_rank(group)
    for r, p in enumerate(ptrs):
        if r != rank:
            cc.ipc_close(p)


def setup_peer_tier(ctx, lend_bytes, device, group=None):
    """E-10 over a ring: each rank lends `lend_bytes` of its HBM to the previous rank and evicts
    into the next rank's loan (cc_set_peer_tier).  Returns (lent buffer, mapped addresses) —
    keep both alive until every rank's last cc_execute returned (barrier), then close_buffers."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lent = torch.empty(int(lend_bytes), dtype=torch.uint8, device=device)
    ptrs = exchange_buffers(lent, group)
    ctx.set_peer_tier(ptrs[(rank + 1) % world], int(lend_bytes))
    return lent, ptrs


def share_leaves(ctx, host_leaves, device, group=None):
    """E-11 under a TREES split (rank = TREES part): the owner of each leaf (cc_leaf_owners)
    copies it host -> its HBM once; every rank then points each leaf at the owner's copy
    (cc_set_leaf_peer: a peer copy over NVLink, or a local device copy for its own leaves).
    host_leaves: {leaf id: pinned host tensor of the full leaf}.  Returns (peer leaf ids for
    cc_schedule's peer_leaves, own staging buffer, mapped addresses); the caller keeps the
    buffers alive, and times the staging (H2D of the owned leaves) as part of the run."""
    rank = dist.get_rank(group)
    owners = ctx.leaf_owners()
    mine = sorted(u for u, o in owners.items() if o == rank)
    offs, total = {}, 0
    for u in mine:
        offs[u] = total
        total += (host_leaves[u].numel() * host_leaves[u].element_size() + 255) // 256 * 256
    buf = torch.empty(max(total, 256), dtype=torch.uint8, device=device)
    for u in mine:
        n = host_leaves[u].numel() * host_leaves[u].element_size()
        buf[offs[u]:offs[u] + n].view(host_leaves[u].dtype).copy_(host_leaves[u], non_blocking=True)
    all_offs = [None] * dist.get_world_size(group)
    dist.all_gather_object(all_offs, offs, group=group)
    torch.cuda.synchronize(device)
    ptrs = exchange_buffers(buf, group)
    dist.barrier(group)                     # every owner's copies have landed
    for u, o in owners.items():
        ctx.set_leaf_peer(u, ptrs[o] + all_offs[o][u], host_leaves[u].numel() * host_leaves[u].element_size())
    return sorted(owners), buf, ptrs
