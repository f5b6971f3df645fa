"""O6 — exact minimum peak memory over all valid schedules.

TEST INFRASTRUCTURE (see oracle/__init__.py).  The problem statement: "find a
sequential schedule of the contraction DAG that minimizes the peak memory,
i.e., max_i M_i" under the §II-C model.

Two exact methods, used only on tiny DAGs:
  brute_force_peak : every linear extension, each replayed by memory.simulate
  dp_peak          : min-max DP over completed-contraction bitsets; the resident
                     set after a step is a function of the completed set alone
                     (a leaf is resident iff some but not all of its parents are
                     done; a non-leaf iff it is done and some parent is not).
"""
import itertools

from .memory import simulate, check_schedule


def brute_force_peak(dag, limit=8):
    contr = dag.contractions()
    if len(contr) > limit:
        raise ValueError("too many contractions for brute force")
    best = None
    best_order = None
    for perm in itertools.permutations(contr):
        if check_schedule(dag, list(perm)):
            continue
        p = simulate(dag, list(perm))["peak"]
        if best is None or p < best:
            best, best_order = p, list(perm)
    return best, best_order


def dp_peak(dag, limit=16):
    contr = dag.contractions()
    n = len(contr)
    if n > limit:
        raise ValueError("too many contractions for the DP")
    idx = {u: i for i, u in enumerate(contr)}
    nodes = dag.nodes
    need = []
    for u in contr:
        m = 0
        for c in nodes[u].child:
            if c in idx:
                m |= 1 << idx[c]
        need.append(m)

    def mem(mask):
        total = 0
        for u, nd in nodes.items():
            if nd.child:
                done = bool(mask >> idx[u] & 1)
                if done and any(not (mask >> idx[p] & 1) for p in nd.parents):
                    total += nd.size
            else:
                ps = [mask >> idx[p] & 1 for p in nd.parents]
                if any(ps) and not all(ps):
                    total += nd.size
        return total

    full = (1 << n) - 1
    INF = float("inf")
    best = [INF] * (1 << n)
    back = [-1] * (1 << n)
    best[0] = 0
    for mask in range(1 << n):           # masks in increasing order: subsets first
        if best[mask] == INF:
            continue
        for i in range(n):
            if mask >> i & 1 or (need[i] & mask) != need[i]:
                continue
            nm = mask | 1 << i
            v = max(best[mask], mem(nm))
            if v < best[nm]:
                best[nm] = v
                back[nm] = i
    order = []
    m = full
    while m:
        i = back[m]
        order.append(contr[i])
        m &= ~(1 << i)
    order.reverse()
    return best[full], order
