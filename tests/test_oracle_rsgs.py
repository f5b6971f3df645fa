"""Pins of the RS-GS-like baseline (oracle/rsgs.py, readings R-1..R-4).

- hand-derived chains and orders on D* and F1 (Jaccard values written out below)
- disjoint trees -> tree-id order (all similarities 0, R-2 tie rule)
- a near-identical pair is chained together even when ids separate it
- greedy maximality re-derived by brute force (every pair's Jaccard as an exact Fraction,
  full scan) on random DAGs — independent of the inverted-index shortcut in the oracle
- validity of every order under the §II-C checker; optimum <= RS-GS peak
"""
from fractions import Fraction

import pytest

from synth import dags
from oracle.dag import Dag
from oracle.memory import simulate, check_schedule
from oracle import rsgs, optimum

D = dict(zip("abcdefgh", range(8)))
F = dict(a=0, b=1, e=2, f=3, g=4, h=5, l=6)


def test_dstar_chain_and_order():
    # T0={f,a,b}  T1={g,a,e,b,c}  T2={h,d,e,b,c}
    # J(T0,T1) = |{a,b}|/|{a,b,c,e,f,g}| = 2/6 > J(T0,T2) = |{b}|/|{a,b,c,d,e,f,h}| = 1/7
    dag = Dag(dags.fixture_dstar())
    assert rsgs.tree_chain(dag) == [0, 1, 2]
    order = rsgs.schedule(dag)
    # T0: f;  T1 post-order from g=(a,e): e=(b,c), g;  T2: h=(d,e) with e done
    assert order == [D[c] for c in "fegh"]
    assert simulate(dag, order)["residency"] == [0, 2, 2, 1, 0]


def test_f1_chain_and_order():
    # T0 = g-tree {g,e,a,b,l}, T1 = h-tree {h,e,a,b,l}, T2 = f-tree {f,a,b}
    # J(T0,T1) = 4/6 > J(T0,T2) = 2/6
    dag = Dag(dags.fixture_f1())
    assert rsgs.tree_chain(dag) == [0, 1, 2]
    order = rsgs.schedule(dag)
    assert order == [F[c] for c in "eghf"]
    assert simulate(dag, order)["residency"] == [0, 2, 3, 2, 0]


def _workload(trees):
    """trees: list of (root_id, [(id, a, b), ...]) over shared meson leaves 0..9."""
    w = dags.Workload("t", 1, 2, 1)
    used = sorted({x for _, ops in trees for (_, a, b) in ops for x in (a, b) if x < 10})
    w.nodes = [(i, dags.LEAF_M, -1, -1, 0) for i in used]
    w.trees = []
    for tid, (root, ops) in enumerate(trees):
        for (i, a, b) in ops:
            w.nodes.append((i, dags.TR_MM if i == root else dags.MM1, a, b, 0))
        w.trees.append((tid, root))
    return w


def test_disjoint_trees_in_id_order():
    w = _workload([(100, [(100, 0, 1)]), (101, [(101, 2, 3)]), (102, [(102, 4, 5)])])
    dag = Dag(w)
    assert rsgs.tree_chain(dag) == [0, 1, 2]
    assert rsgs.schedule(dag) == [100, 101, 102]


def test_similar_pair_chained_across_ids():
    # tree 0 = TR(MM1(0,1), MM1(2,3)); tree 1 disjoint; tree 2 shares MM1(0,1) and leaves 2,3
    w = _workload([(100, [(10, 0, 1), (11, 2, 3), (100, 10, 11)]),
                   (101, [(101, 6, 7)]),
                   (102, [(12, 3, 2), (102, 10, 12)])])
    dag = Dag(w)
    assert rsgs.tree_chain(dag) == [0, 2, 1]
    assert rsgs.schedule(dag) == [10, 11, 100, 12, 102, 101]


def _brute_chain(dag):
    members = {t: set(dag.trees[t][1]) for t in dag.tree_ids}
    left = sorted(dag.tree_ids)
    chain = [left.pop(0)]
    while left:
        prev = members[chain[-1]]
        sims = [(Fraction(len(prev & members[t]), len(prev | members[t])), -t) for t in left]
        best = max(sims)
        t = -best[1]
        chain.append(t)
        left.remove(t)
    return chain


@pytest.mark.parametrize("seed", range(40))
def test_greedy_chain_matches_brute_force(seed):
    w = dags.random_dag(seed, n_leaves=7, n_trees=7, max_ops_per_tree=4, share_p=0.6, typed=(seed % 2 == 0))
    dag = Dag(w)
    assert rsgs.tree_chain(dag) == _brute_chain(dag)
    order = rsgs.schedule(dag)
    assert check_schedule(dag, order) == []
    assert sorted(order) == sorted(u for u, n in dag.nodes.items() if n.child)


@pytest.mark.parametrize("seed", range(12))
def test_optimum_bounds_rsgs(seed):
    w = dags.random_dag(seed, n_leaves=5, n_trees=4, max_ops_per_tree=3, share_p=0.6)
    dag = Dag(w)
    if len(dag.contractions()) > 14:
        pytest.skip("too large for the DP")
    opt = optimum.dp_peak(dag)[0]
    assert opt <= simulate(dag, rsgs.schedule(dag))["peak"]


def test_configs_valid():
    for w in (dags.config_c2(N=8, Lt=1), dags.config_c4(N=4, Lt=1, S=2, n_trees=300)):
        dag = Dag(w)
        order = rsgs.schedule(dag)
        assert check_schedule(dag, order) == []
