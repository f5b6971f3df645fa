"""Multi-GPU partition (the paper lists partitioning as future
work).  TEST INFRASTRUCTURE (see oracle/__init__.py).

TIME: part p of n owns time slices [p*Lt//n, (p+1)*Lt//n) — every op is per-slice.
TREES: trees in tree-scheduler selection order (O4); tree weight = flops/8 of the
contractions first executed while processing it (MM1 Lt N^3, BM1/BB2 Lt S N^4, TR Lt N^2,
BB1/BT2 Lt S N^5, BB3 Lt S N^3;
abstract DAGs: 1 per contraction); tree i with prefix weight P_i, weight w_i, total W goes
to part min(n-1, floor(n (2 P_i + w_i) / (2 W))).
"""
from synth.dags import MM1, BM1, BB2, TR_MM, BB1, BT2, BB3, Workload
from .dag import Dag
from . import tree as tree_sched


def time_range(Lt, n_parts, part):
    return (part * Lt // n_parts, (part + 1) * Lt // n_parts)


def _weight(dag, u):
    n = dag.nodes[u]
    if n.op in (MM1,):
        return dag.Lt * dag.N ** 3
    if n.op in (BM1, BB2):
        return dag.Lt * dag.S * dag.N ** 4
    if n.op == TR_MM:
        return dag.Lt * dag.N ** 2
    if n.op in (BB1, BT2):
        return dag.Lt * dag.S * dag.N ** 5
    if n.op == BB3:
        return dag.Lt * dag.S * dag.N ** 3
    return 1


def tree_parts(dag, n_parts):
    """{tree_id: part} for a TREES split."""
    s = tree_sched.TreeScheduler(dag)
    order = s.run()
    sel = s.tree_order
    owner = {}
    for t in sel:
        for u in dag.trees[t][1]:
            owner.setdefault(u, t)
    w = {t: 0 for t in sel}
    for u in order:
        w[owner[u]] += _weight(dag, u)
    W = sum(w.values())
    parts = {}
    P = 0
    for t in sel:
        p = (n_parts * (2 * P + w[t])) // (2 * W) if W > 0 else 0
        parts[t] = min(n_parts - 1, p)
        P += w[t]
    return parts


def sub_workload(w, keep_trees):
    """The workload restricted to some trees (closure of their roots; terms of those trees)."""
    dag = Dag(w)
    keep = set(keep_trees)
    nodes = set()
    for t in keep:
        nodes |= dag.trees[t][1]
    return Workload(w.name + "_part", w.Lt, w.N, w.S,
                    nodes=[n for n in w.nodes if n[0] in nodes],
                    trees=[t for t in w.trees if t[0] in keep],
                    terms=[x for x in w.terms if x[1] in keep],
                    data_seed=w.data_seed, leaf_mode=w.leaf_mode)
