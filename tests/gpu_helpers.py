"""Helpers for the -m gpu parity tests: run a synth Workload through the C ABI."""
import numpy as np

from oracle import values
from oracle.dag import Dag


def pinned_from(v):
    import torch
    h = torch.empty(v.size * 2, dtype=torch.float64, pin_memory=True)
    h.numpy()[:] = np.ascontiguousarray(v).view(np.float64).ravel()
    return h


def device_from(v):
    import torch
    return torch.from_numpy(np.ascontiguousarray(v).view(np.float64).ravel().copy()).cuda()


def to_numpy_c(t, shape):
    a = t.detach().cpu().numpy().view(np.complex128)
    return a.reshape(shape)


def run_gpu(w, algo=None, cap=0, flags=0, device_leaves=False, arena_mb=256, leaf_fn=None, ctx=None,
            part=None, evict_next_use=False, options=None, peer_cap=0, peer_leaves=(), peer_tier_mb=0):
    """Returns (ctx, roots{tree: [Lt]}, corr{c: [Lt]}, plan stats, exec stats).
    options: executor options for cc_set_options (cc.h cc_options), e.g. {"trace_fusion": 1}.
    peer_cap / peer_leaves / peer_tier_mb: the peer-HBM tier (E-10, E-11) with its region and the
    peer-homed leaves' copies as buffers on this GPU (a loopback stand-in for a peer GPU's HBM)."""
    import torch
    from paper_2511_02257_b200 import cc
    dag = Dag(w)
    if ctx is None:
        arena = torch.empty(arena_mb << 20, dtype=torch.uint8, device="cuda")
        ctx = cc.Context(0, arena)
    if options:
        ctx.set_options(**options)
    ctx.load_workload(w)
    if part is not None:
        if part[0] == "grid":               # ("grid", n_tree_parts, n_time_parts, part)
            ctx.partition_grid(*part[1:])
        else:
            ctx.partition(*part)
    order, st = ctx.schedule(cc.CC_TREE if algo is None else algo, cap_bytes=cap, evict_next_use=evict_next_use,
                             peer_cap_bytes=peer_cap, peer_leaves=peer_leaves)
    keep = []
    if peer_tier_mb:
        tier = torch.empty(peer_tier_mb << 20, dtype=torch.uint8, device="cuda")
        keep.append(tier)
        ctx.set_peer_tier(tier)
    Lt_part = w.Lt
    t0 = 0
    if part is not None:
        t0, t1 = ctx.part_time_range()
        Lt_part = t1 - t0
    for u, n in dag.nodes.items():
        if n.child:
            continue
        v = leaf_fn(u, n.op) if leaf_fn else values.synthetic_leaf(w, u, n.op)
        if hasattr(v, "data_ptr"):          # a ready pinned host tensor of the full leaf
            assert not device_leaves and part is None
            keep.append(v)
            ctx.set_leaf(u, v)
            continue
        if u in peer_leaves:
            d = device_from(v)                     # the full leaf, as a peer rank would hold it
            keep.append(d)
            ctx.set_leaf_peer(u, d)
            continue
        if device_leaves:
            d = device_from(v[t0:t0 + Lt_part])
            keep.append(d)
            ctx.set_leaf_device(u, d)
        else:
            h = pinned_from(v)
            keep.append(h)
            ctx.set_leaf(u, h)
    ex = ctx.execute(flags)
    if flags & 1:
        ex = ctx.execute(flags)     # a graph replay after the capturing run
    ctx._leaf_buffers = keep
    trees = ctx.part_trees()
    roots = {t: ctx.root_value(t, Lt_part) for t in trees}
    corr = {}
    _, n_corr, ids = ctx.correlator_device_ptr()
    for c in ids:
        corr[c] = ctx.correlator(c, Lt_part)
    return ctx, roots, corr, st, ex


def assert_roots_close(got, want, rel=1e-10):
    worst = 0.0
    for t, w in want.items():
        g = got[t]
        err = np.max(np.abs(g - w) / np.maximum(np.abs(w), 1e-300))
        worst = max(worst, float(err))
    assert worst <= rel, "worst relative root error %g > %g" % (worst, rel)
    return worst


def assert_corr_close(dag, roots_oracle, got, want, rel=1e-10):
    scale = values.term_scale(dag, roots_oracle)
    for c, w in want.items():
        assert np.all(np.abs(got[c] - w) <= rel * scale[c] + 1e-300), c
