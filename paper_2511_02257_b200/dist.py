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


class SharedLeaves:
    """E-11 under a TREES split (rank = TREES part): every leaf is held in the HBM of its owner
    (cc_leaf_owners), which loads it over PCIe once per run (stage()); every rank points each
    leaf at the owner's copy (cc_set_leaf_peer: a peer copy over NVLink, or a local device copy
    for its own leaves) and schedules with peer_leaves = ids.
    leaf_bytes: {leaf id: bytes of the full leaf}; host_owned: {leaf id: pinned host tensor}
    for the leaves this rank owns.  Keep the object alive until every rank's last cc_execute
    returned (barrier), then close()."""

    def __init__(self, ctx, leaf_bytes, host_owned, device, group=None):
        self.group = group
        rank = dist.get_rank(group)
        owners = ctx.leaf_owners()
        self.mine = sorted(u for u, o in owners.items() if o == rank)
        self.offs, total = {}, 0
        for u in self.mine:
            self.offs[u] = total
            total += (leaf_bytes[u] + 255) // 256 * 256
        self.buf = torch.empty(max(total, 256), dtype=torch.uint8, device=device)
        self.host = host_owned
        all_offs = [None] * dist.get_world_size(group)
        dist.all_gather_object(all_offs, self.offs, group=group)
        self.ptrs = exchange_buffers(self.buf, group)
        for u, o in owners.items():
            ctx.set_leaf_peer(u, self.ptrs[o] + all_offs[o][u], leaf_bytes[u])
        self.ids = sorted(owners)

    def stage(self):
        """Owners copy their leaves host -> HBM (the run's only leaf PCIe traffic; current
        stream); returns the bytes copied.  Ends with a barrier: every owner's copies landed."""
        n = 0
        for u in self.mine:
            h = self.host[u]
            nb = h.numel() * h.element_size()
            self.buf[self.offs[u]:self.offs[u] + nb].view(h.dtype).copy_(h, non_blocking=True)
            n += nb
        torch.cuda.synchronize()
        dist.barrier(self.group)
        return n

    def close(self):
        close_buffers(self.ptrs, self.group)
