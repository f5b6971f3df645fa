"""O3 — sibling scheduler, Alg. 1-3 (§III-A).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Follows the pseudocode line by
line with the pins of DESIGN.md §Readings:
  S-1 "random leaf" (Alg. 1 l.4) = lowest-id WAITING leaf
  S-2 FIFO within each queue Q_i
  S-3 u.parents iterated in ascending id (Alg. 2 l.13)
  S-4 prop-down is immediate and depth first, left operand then right (Alg. 3 l.9-10)
  S-6 prop-down may fire once per parent; the WAITING guard absorbs repeats
  G-6 the schedule is the contraction order; leaf loads are lazy in O2/O5.
"""
from collections import deque

WAITING, QUEUED, INMEM, RELEASED = "WAITING", "QUEUED", "INMEM", "RELEASED"


class StuckError(Exception):
    pass


def schedule(dag, trace=None):
    """Alg. 1 SB-SCHEDULER.  Returns the contraction order (list of node ids).
    `trace`, if a list, receives ("load"|"contract", id) events in order."""
    nodes = dag.nodes
    # fields of P:263-286
    rs = {u: len(n.parents) for u, n in nodes.items()}      # remaining successors
    rp = {u: len(n.child) for u, n in nodes.items()}        # remaining predecessors
    state = {u: WAITING for u in nodes}
    q = max(n.rank for n in nodes.values())
    queues = [None] + [deque() for _ in range(q)]           # Q_1..Q_q
    leaves = [u for u in dag.ids if not nodes[u].child]     # ascending id (S-1)
    leaf_cursor = [0]
    order = []
    n_contr = len(dag.contractions())
    calls = {"process": 0}

    def sb_process(u):                                      # Alg. 2
        calls["process"] += 1
        n = nodes[u]
        if n.child:
            order.append(u)                                 # l.2 perform the contraction
            if trace is not None:
                trace.append(("contract", u))
        elif trace is not None:
            trace.append(("load", u))                       # l.4 bring the tensor to memory
        state[u] = INMEM                                    # l.5
        if n.child:                                         # l.6-12 releasable nodes
            for v in n.child:
                rs[v] -= 1
                if rs[v] == 0:
                    state[v] = RELEASED
            if not n.parents:                               # ROOT (l.11-12)
                state[u] = RELEASED
        for v in n.parents:                                 # l.13-21, ascending id (S-3)
            rp[v] -= 1
            if rp[v] == 1:
                a, b = nodes[v].child
                w = b if a == u else a                      # the sibling of u under v
                if state[w] == WAITING:
                    sb_prop_down(w)
            elif rp[v] == 0:
                queues[nodes[v].rank].append(v)             # ENQUEUE(Q_{v.rank}, v)
                state[v] = QUEUED

    def sb_prop_down(u):                                    # Alg. 3
        if state[u] != WAITING:
            return
        if not nodes[u].child:
            sb_process(u)
            return
        left, right = nodes[u].child
        sb_prop_down(left)
        sb_prop_down(right)

    while len(order) < n_contr:                             # Alg. 1
        i = q
        while i >= 1 and not queues[i]:
            i -= 1
        if i == 0:                                          # all queues empty
            while leaf_cursor[0] < len(leaves) and state[leaves[leaf_cursor[0]]] != WAITING:
                leaf_cursor[0] += 1
            if leaf_cursor[0] == len(leaves):
                raise StuckError("no WAITING leaf and all queues empty")
            u = leaves[leaf_cursor[0]]
        else:
            u = queues[i].popleft()                         # FIFO (S-2)
        sb_process(u)
    schedule.last_calls = calls["process"]
    return order
