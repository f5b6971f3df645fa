"""Multi-GPU partition (the paper lists partitioning as future
work).  TEST INFRASTRUCTURE (see oracle/__init__.py).

TIME: part p of n owns time slices [p*Lt//n, (p+1)*Lt//n) — every op is per-slice.
TREES (reading M-1, round 2): trees in tree-scheduler selection order (O4), cut into n
contiguous chunks; a chunk's work is what its part executes: flops/8 of the distinct
contractions in the union of its trees' closures, shared nodes replicated (MM1 Lt N^3,
BM1/BB2 Lt S N^4, TR Lt N^2, BB1/BT2 Lt S N^5, BB3 Lt S N^3; abstract DAGs: 1 per
contraction).  The cut minimises the largest chunk's work: T* = the smallest T for which the
first-fit cut (extend the current chunk while its work stays <= T) needs at most n chunks
(exact for min-max contiguous partitions: chunk work only grows when a chunk is extended);
the parts are that first-fit cut at T*; while there are fewer than n chunks, the chunk of
largest work with at least two trees (lowest index on ties) is split in half by tree count.
(Round 1 balanced first-execution work, which ignores the replicas: on c4 at 8 parts the
largest part executed 1.59x the mean.)
GRID (reading M-2): n_tree x n_time parts; part p is TREES part p // n_time restricted to
TIME slices of part p % n_time (every op is per-slice, so the two splits compose).
Replication (SURVEY §8(d) "replicas ... counted as overhead and reported", reading M-3): the
owner of a node is the part of the first selected tree containing it; a part's replicated
work / leaf bytes are those of its contractions / leaves owned by another part.
Leaf owners (reading E-11): the same owner rule names the rank that loads a shared leaf over
PCIe; the other parts using it read that copy over NVLink.
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


def _owners(dag):
    """(contraction order, tree selection order, {node: first selected tree containing it})."""
    s = tree_sched.TreeScheduler(dag)
    order = s.run()
    sel = s.tree_order
    owner = {}
    for t in sel:
        for u in dag.trees[t][1]:
            owner.setdefault(u, t)
    return order, sel, owner


def _closure_contractions(dag, t):
    return [u for u in dag.trees[t][1] if dag.nodes[u].child]


def chunk_work(dag, trees):
    """Work (flops/8) of the distinct contractions in the union of the trees' closures."""
    seen = set()
    for t in trees:
        seen.update(_closure_contractions(dag, t))
    return sum(_weight(dag, u) for u in seen)


def _first_fit(dag, sel, T):
    """Chunks of the first-fit cut at work bound T, or None if one tree alone exceeds T."""
    out, cur, seen, w = [], [], set(), 0
    for t in sel:
        mem = _closure_contractions(dag, t)
        add = sum(_weight(dag, u) for u in mem if u not in seen)
        if cur and w + add > T:
            out.append(cur)
            cur, seen, w = [], set(), 0
            add = sum(_weight(dag, u) for u in mem)
        if add > T:
            return None
        cur.append(t)
        seen.update(mem)
        w += add
    if cur:
        out.append(cur)
    return out


def tree_parts(dag, n_parts):
    """{tree_id: part} for a TREES split (reading M-1, module docstring)."""
    _, sel, _ = _owners(dag)
    lo = max([chunk_work(dag, [t]) for t in sel] + [0])
    hi = chunk_work(dag, sel)
    while lo < hi:                                  # smallest T with <= n first-fit chunks
        mid = (lo + hi) // 2
        c = _first_fit(dag, sel, mid)
        if c is not None and len(c) <= n_parts:
            hi = mid
        else:
            lo = mid + 1
    chunks = _first_fit(dag, sel, lo) if sel else []
    while len(chunks) < n_parts:
        cand = [(chunk_work(dag, c), -k) for k, c in enumerate(chunks) if len(c) >= 2]
        if not cand:
            break
        k = -max(cand)[1]
        c = chunks[k]
        h = len(c) // 2
        chunks[k:k + 1] = [c[:h], c[h:]]
    return {t: p for p, c in enumerate(chunks) for t in c}


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


def grid_part(n_tree, n_time, part):
    """GRID part index -> (TREES part, TIME part) (reading M-2)."""
    return part // n_time, part % n_time


def part_stats(w, n_parts, part, n_time=1):
    """Work (flops / 8, weights of _weight at this part's slice count) and leaf bytes of one
    part of a TREES (n_time == 1) or GRID split, with the replicated share (reading M-3)."""
    dag = Dag(w)
    pt, ptm = grid_part(n_parts, n_time, part)
    t0, t1 = time_range(w.Lt, n_time, ptm)
    parts = tree_parts(dag, n_parts)
    _, _, owner = _owners(dag)
    keep = [t for t in dag.tree_ids if parts[t] == pt]
    sub = Dag(sub_workload(w, keep))
    scale = Dag(Workload(w.name, t1 - t0, w.N, w.S, nodes=w.nodes, trees=w.trees, terms=w.terms))
    st = dict(n_trees=len(keep), n_contr=0, work=0, replicated_work=0, leaf_bytes=0, replicated_leaf_bytes=0)
    for u, n in sub.nodes.items():
        mine = parts[owner[u]] == pt
        if n.child:
            wu = _weight(scale, u)
            st["n_contr"] += 1
            st["work"] += wu
            st["replicated_work"] += 0 if mine else wu
        else:
            b = n.size * (t1 - t0) // w.Lt
            st["leaf_bytes"] += b
            st["replicated_leaf_bytes"] += 0 if mine else b
    return st


def leaf_owners(w, n_parts):
    """{leaf id: part that loads it over PCIe} for a TREES split (reading E-11)."""
    dag = Dag(w)
    parts = tree_parts(dag, n_parts)
    _, _, owner = _owners(dag)
    return {u: parts[owner[u]] for u, n in dag.nodes.items() if not n.child and u in owner}
