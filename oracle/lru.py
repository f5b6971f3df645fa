"""O5 — capacity-limited device plan with LRU eviction to host.

TEST INFRASTRUCTURE (see oracle/__init__.py).

MemHC's "pre-protected LRU" is named, not defined, in the paper; this
follows DESIGN.md readings E-1..E-8:
  E-1 before c_i: need = sum of non-resident operand sizes + output size; while
      used + need > cap evict the least-recently-used resident tensor that is not
      an operand of c_i.  Infeasible if operands + output > cap.
  E-2 LRU clock: a global counter, one tick per touch; at c_i the operands are
      touched in (left, right) order (a fetch is a touch), then the output.
  E-3 evicting a leaf: 1 eviction, no D2H (the host copy is the caller's).
  E-4 evicting an intermediate: 1 eviction + D2H on its FIRST eviction; the host
      copy is kept until release, so later evictions of it are clean drops.
  E-5 #transfers = h2d_count + d2h_count.
  E-8 tensors nothing depends on are released at once (never "evicted").
Leaves are fetched lazily at first use (G-6).  Release follows §II-C.

policy="next_use" (reading E-9; SURVEY f3 "Belady/next-use eviction, since the whole
schedule is known offline"): the victim is the resident non-operand of c_i whose next use
(the first later contraction that reads it) is farthest away; ties go to the least recently
used (E-2 clock).  Everything else (E-1..E-8) is unchanged.

Peer-HBM tier (readings E-10, E-11; SURVEY f3 "NVLink peer-HBM eviction tier + cross-GPU
leaf sharing", attacking the PCIe bottleneck of P:70-72):
  E-10 a victim without an off-device copy (an intermediate at its first eviction, or a leaf
       whose home is the host) is copied to a peer GPU's HBM ("P2P_OUT", NVLink) when the
       peer tier's remaining capacity (peer_cap bytes) holds it; otherwise E-3 / E-4 apply
       unchanged (DROP for a leaf, D2H for an intermediate).  The peer copy, like the host copy
       of E-4, is kept until the tensor is released, so later evictions of it are clean DROPs
       and its re-fetches are "P2P_IN" (NVLink) instead of H2D (PCIe).  Peer-tier bytes are
       freed at release.  No tensor moves between the peer tier and the host.
  E-11 a leaf in `peer_leaves` has its home copy in a peer GPU's HBM (cross-GPU leaf sharing:
       one rank loads it over PCIe, the others read that copy): each of its fetches is a
       P2P_IN, an eviction of it is a DROP, and it never occupies this rank's peer tier.
With peer_cap = 0 and no peer leaves the plan is exactly the E-1..E-9 plan.
"""


class InfeasibleError(Exception):
    pass


def _next_uses(dag, order):
    """uses[x] = ascending list of the steps i whose contraction reads x."""
    uses = {}
    for i, u in enumerate(order):
        for x in dag.nodes[u].child:
            uses.setdefault(x, []).append(i)
    return uses


def plan(dag, order, cap=None, policy="lru", peer_cap=0, peer_leaves=()):
    """Replay `order` on a device of `cap` bytes (None or <= 0: unbounded); policy "lru"
    (E-1) or "next_use" (E-9); peer tier of `peer_cap` bytes (E-10) and leaves whose home is a
    peer GPU (E-11).

    Returns dict: ops [(kind, node)], kinds in {"D2H","DROP","H2D","CONTRACT","FREE"}
    ("D2H" = eviction with a copy to host, "DROP" = eviction without copy),
    evictions, h2d_count, d2h_count, h2d_bytes, d2h_bytes, peak (device bytes after
    each step's releases), transient_peak (device bytes right after the output is
    produced), host_peak_bytes (host copies of evicted intermediates), used [per step];
    peer tier: kinds "P2P_OUT" (eviction copied to the peer tier) and "P2P_IN" (fetch from a
    peer), p2p_out_count / p2p_out_bytes / p2p_in_count / p2p_in_bytes, peer_peak_bytes.
    """
    if cap is not None and cap <= 0:
        cap = None
    nodes = dag.nodes
    remaining = {u: len(n.parents) for u, n in nodes.items()}
    resident = set()
    host_copy = set()
    lru = {}
    clock = 0
    used = 0
    host_bytes = 0
    st = dict(evictions=0, h2d_count=0, d2h_count=0, h2d_bytes=0, d2h_bytes=0,
              peak=0, transient_peak=0, host_peak_bytes=0,
              p2p_out_count=0, p2p_out_bytes=0, p2p_in_count=0, p2p_in_bytes=0, peer_peak_bytes=0)
    peer_home = set(peer_leaves)
    for x in peer_home:
        assert not nodes[x].child, "E-11: only leaves have a peer home"
    peer_copy = set()                   # tensors with a copy in this rank's peer tier (E-10)
    peer_used = 0
    ops = []
    used_trace = [0]
    uses = _next_uses(dag, order)
    ptr = {x: 0 for x in uses}          # uses[x][ptr[x]] = next step reading x

    def next_use(x):
        return uses[x][ptr[x]]

    for i, u in enumerate(order):
        n = nodes[u]
        operands = list(n.child)
        work = sum(nodes[x].size for x in operands) + n.size
        if cap is not None and work > cap:
            raise InfeasibleError("contraction %d needs %d bytes > cap %d" % (u, work, cap))
        need = sum(nodes[x].size for x in operands if x not in resident) + n.size
        while cap is not None and used + need > cap:          # E-1
            cands = [x for x in resident if x not in operands]
            if policy == "next_use":                              # E-9: farthest next use
                victim = max(cands, key=lambda x: (next_use(x), -lru[x]))
            else:
                victim = min(cands, key=lambda x: lru[x])
            st["evictions"] += 1
            size = nodes[victim].size
            # E-10: stash candidates are the victims with no copy outside the device except
            # the caller's host copy of a leaf (an intermediate's host copy comes from E-4)
            stash = victim not in peer_copy and victim not in peer_home and victim not in host_copy
            if stash and peer_used + size <= peer_cap:             # E-10: copy to the peer tier
                st["p2p_out_count"] += 1
                st["p2p_out_bytes"] += size
                peer_copy.add(victim)
                peer_used += size
                st["peer_peak_bytes"] = max(st["peer_peak_bytes"], peer_used)
                ops.append(("P2P_OUT", victim))
            elif nodes[victim].child and stash:                    # E-4 first eviction
                st["d2h_count"] += 1
                st["d2h_bytes"] += size
                host_copy.add(victim)
                host_bytes += size
                st["host_peak_bytes"] = max(st["host_peak_bytes"], host_bytes)
                ops.append(("D2H", victim))
            else:                                                  # E-3 / clean E-4
                ops.append(("DROP", victim))
            resident.discard(victim)
            used -= nodes[victim].size
        for x in operands:                                         # this step's use is consumed
            ptr[x] += 1
        for x in operands:                                         # fetch + touch (E-2)
            if x not in resident:
                if x in peer_copy or x in peer_home:               # E-10 / E-11: over NVLink
                    st["p2p_in_count"] += 1
                    st["p2p_in_bytes"] += nodes[x].size
                    ops.append(("P2P_IN", x))
                else:
                    st["h2d_count"] += 1
                    st["h2d_bytes"] += nodes[x].size
                    ops.append(("H2D", x))
                resident.add(x)
                used += nodes[x].size
            clock += 1
            lru[x] = clock
        resident.add(u)                                            # output
        used += n.size
        clock += 1
        lru[u] = clock
        ops.append(("CONTRACT", u))
        st["transient_peak"] = max(st["transient_peak"], used)
        for x in operands:                                         # release at last use
            remaining[x] -= 1
            if remaining[x] == 0:
                resident.discard(x)
                used -= nodes[x].size
                if x in host_copy:
                    host_copy.discard(x)
                    host_bytes -= nodes[x].size
                if x in peer_copy:
                    peer_copy.discard(x)
                    peer_used -= nodes[x].size
                ops.append(("FREE", x))
        if remaining[u] == 0:                                      # ROOT: released at once
            resident.discard(u)
            used -= n.size
            ops.append(("FREE", u))
        st["peak"] = max(st["peak"], used)
        used_trace.append(used)
    assert used == 0 and not resident and host_bytes == 0 and peer_used == 0
    st["ops"] = ops
    st["used"] = used_trace
    st["transfers"] = st["h2d_count"] + st["d2h_count"]
    return st
