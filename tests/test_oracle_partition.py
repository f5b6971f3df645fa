"""Pins of oracle/partition.py (readings M-1..M-3; partitioning is future
work in the paper) against hand-derived parts (D*) and properties the rule must satisfy:
contiguity in tree-scheduler selection order, non-empty parts, and a largest part work
(replicas included) equal to the brute-force minimum over all contiguous cuts."""
import itertools

import pytest

from synth import dags
from oracle import partition, tree as tree_sched
from oracle.dag import Dag


def _selection(dag):
    s = tree_sched.TreeScheduler(dag)
    s.run()
    return s.tree_order


def test_dstar_hand_parts():
    """D* (Table I DAG, unit weights: abstract contractions weigh 1).  The tree scheduler selects
    T0 (f), T1 (g), T2 (h) (SURVEY §8(c) O4 hand trace).  Closure contractions: T0 {f},
    T1 {e, g}, T2 {e, h}.  n = 2: bound 2 cuts [T0] | [T1] | [T2] (T0 + T1 would be 3) — three
    chunks; bound 3: [T0, T1] (work 3) | [T2] (T2 adds h only while e is in the chunk, but
    4 > 3 cuts it; alone it weighs 2) — two chunks, so T* = 3 and the parts are {0, 0, 1}.
    n = 3: bound 2 gives the three singletons.  n = 1: one chunk."""
    dag = Dag(dags.fixture_dstar())
    assert _selection(dag) == [0, 1, 2]
    assert partition.tree_parts(dag, 2) == {0: 0, 1: 0, 2: 1}
    assert partition.tree_parts(dag, 3) == {0: 0, 1: 1, 2: 2}
    assert partition.tree_parts(dag, 1) == {0: 0, 1: 0, 2: 0}
    assert partition.chunk_work(dag, [0, 1]) == 3 and partition.chunk_work(dag, [1, 2]) == 3


def _weight(w, op):
    # flops / 8 of one contraction: MM1 Lt N^3, BM1 / BB2 Lt S N^4, TR_MM Lt N^2
    return {dags.MM1: w.Lt * w.N ** 3, dags.BM1: w.Lt * w.S * w.N ** 4, dags.BB2: w.Lt * w.S * w.N ** 4,
            dags.TR_MM: w.Lt * w.N ** 2, dags.OP_X: 1}[op]


def _work(dag, ops, w, trees):
    """Independent restatement: distinct contractions of the trees' closures, weighted."""
    nodes = set()
    for t in trees:
        nodes |= {u for u in dag.trees[t][1] if dag.nodes[u].child}
    return sum(_weight(w, ops[u]) for u in nodes)


@pytest.mark.parametrize("seed", range(25))
@pytest.mark.parametrize("n", [2, 3])
def test_partition_min_max_by_brute_force(seed, n):
    """The parts are contiguous in the selection order, all non-empty, and their largest work
    (replicas included) equals the brute-force minimum over every cut of the selection order
    into n non-empty contiguous chunks."""
    typed = seed % 3 != 0
    w = dags.random_dag(seed, n_leaves=6, n_trees=7, max_ops_per_tree=4, share_p=0.6, typed=typed, N=3, Lt=2)
    dag = Dag(w)
    ops = {x[0]: x[1] for x in w.nodes}
    sel = _selection(dag)
    parts = partition.tree_parts(dag, n)
    seq = [parts[t] for t in sel]
    assert sorted(parts) == sorted(dag.tree_ids)
    assert seq == sorted(seq) and set(seq) == set(range(min(n, len(sel))))
    got = max(_work(dag, ops, w, [t for t in sel if parts[t] == p]) for p in set(seq))
    best = None
    for cuts in itertools.combinations(range(1, len(sel)), min(n, len(sel)) - 1):
        bounds = [0, *cuts, len(sel)]
        m = max(_work(dag, ops, w, sel[bounds[k]:bounds[k + 1]]) for k in range(len(bounds) - 1))
        best = m if best is None else min(best, m)
    assert got == best


def test_dstar_part_stats_and_owners():
    """D*, n = 2: part 0 = T0 u T1 = {f, g, e, a, b, c}, part 1 = T2 = {h, e, d, b, c} (unit
    sizes, unit contraction weights).  Owners = part of the first selected tree containing the
    node: a, b, f -> T0, c, e, g -> T1 (part 0); d, h -> T2 (part 1).  Part 1 replicates the
    contraction e and the leaves b, c."""
    w = dags.fixture_dstar()
    assert partition.part_stats(w, 2, 0) == dict(n_trees=2, n_contr=3, work=3, replicated_work=0, leaf_bytes=3,
                                                 replicated_leaf_bytes=0)
    assert partition.part_stats(w, 2, 1) == dict(n_trees=1, n_contr=2, work=2, replicated_work=1, leaf_bytes=3,
                                                 replicated_leaf_bytes=2)
    assert partition.leaf_owners(w, 2) == {0: 0, 1: 0, 2: 0, 3: 1}


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("n,nt", [(2, 1), (3, 2), (2, 4)])
def test_part_stats_properties(seed, n, nt):
    """Replication by an independent formulation: a node's owner part is the smallest part
    index among the trees whose closure holds it (parts are contiguous along the selection
    order); sum over parts of (work - replicated) = the whole DAG's work; GRID time parts
    split each TREES part's work and leaf bytes exactly by slice count."""
    Lt = 4
    w = dags.random_dag(seed, n_leaves=6, n_trees=9, max_ops_per_tree=4, share_p=0.6, typed=True, N=3, Lt=Lt)
    dag = Dag(w)
    ops = {x[0]: x[1] for x in w.nodes}
    parts = partition.tree_parts(dag, n)
    own = {}
    for t in dag.tree_ids:
        for u in dag.trees[t][1]:
            own[u] = min(own.get(u, n), parts[t])
    W = sum(_weight(w, ops[u]) for u, nd in dag.nodes.items() if nd.child)
    used_leaf_bytes = sum(dag.nodes[u].size for u in own if not dag.nodes[u].child)
    tot_unique, tot_leaf_unique = 0, 0
    for pt in range(n):
        rows = [partition.part_stats(w, n, pt * nt + k, n_time=nt) for k in range(nt)]
        keep = [t for t in dag.tree_ids if parts[t] == pt]
        members = set().union(*[dag.trees[t][1] for t in keep]) if keep else set()
        contr = [u for u in members if dag.nodes[u].child]
        work = sum(_weight(w, ops[u]) for u in contr)
        rep = sum(_weight(w, ops[u]) for u in contr if own[u] != pt)
        lb = sum(dag.nodes[u].size for u in members if not dag.nodes[u].child)
        rlb = sum(dag.nodes[u].size for u in members if not dag.nodes[u].child and own[u] != pt)
        t_slices = [partition.time_range(Lt, nt, k) for k in range(nt)]
        for k, r in enumerate(rows):
            frac = (t_slices[k][1] - t_slices[k][0])
            assert r["n_trees"] == len(keep) and r["n_contr"] == len(contr)
            assert r["work"] * Lt == work * frac and r["replicated_work"] * Lt == rep * frac
            assert r["leaf_bytes"] * Lt == lb * frac and r["replicated_leaf_bytes"] * Lt == rlb * frac
        tot_unique += work - rep
        tot_leaf_unique += lb - rlb
    assert tot_unique == W and tot_leaf_unique == used_leaf_bytes
    lo = partition.leaf_owners(w, n)
    assert lo == {u: p for u, p in own.items() if not dag.nodes[u].child}
