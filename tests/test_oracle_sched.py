"""Pins of oracle O3 (sibling, Alg. 1-3), O4 (tree, Alg. 4-8) and O6 (exact optimum).

- hand traces of both schedulers on D* and F1 (derived by hand from the
  pseudocode; D* reproduces Table I)
- from-scratch gains M - M' == incremental tgain at every selection
- tau + delta = |outAv| after every tree
- exact optimum (DP and brute force) <= every scheduler; schedule validity
- structural claims: single tree -> post-order, disjoint trees do not interleave,
  SB-PROCESS called once per node
"""
import numpy as np
import pytest

from synth import dags
from oracle.dag import Dag
from oracle.memory import simulate, check_schedule
from oracle import sibling, tree, optimum

D = dict(zip("abcdefgh", range(8)))          # D* ids
F = dict(a=0, b=1, e=2, f=3, g=4, h=5, l=6)  # F1 ids


def test_sibling_dstar_emits_S1():
    dag = Dag(dags.fixture_dstar())
    trace = []
    order = sibling.schedule(dag, trace)
    assert order == [D[c] for c in "eghf"]                    # = S1 of Table I
    # loads: a (random leaf = lowest id), b and c via prop-down, d via prop-down of h
    assert [u for (k, u) in trace if k == "load"] == [D["a"], D["b"], D["c"], D["d"]]
    assert simulate(dag, order)["residency"] == [0, 2, 3, 2, 0]


def test_sibling_f1():
    dag = Dag(dags.fixture_f1())
    order = sibling.schedule(dag)
    assert order == [F[c] for c in "eghf"]
    assert simulate(dag, order)["residency"] == [0, 2, 3, 2, 0]


def test_tree_dstar_emits_S2_with_gains():
    dag = Dag(dags.fixture_dstar())
    sel = []
    order = tree.schedule(dag, on_select=lambda t, g: sel.append((t, dict(g))))
    assert order == [D[c] for c in "fegh"]                     # = S2 of Table I
    assert sel == [(0, {0: -2, 1: -3, 2: -2}), (1, {1: 1, 2: 0}), (2, {2: 1})]
    assert simulate(dag, order)["residency"] == [0, 2, 2, 1, 0]


def test_tree_f1():
    dag = Dag(dags.fixture_f1())
    sel = []
    order = tree.schedule(dag, on_select=lambda t, g: sel.append((t, dict(g))))
    assert [t for t, _ in sel] == [2, 0, 1]
    assert sel[0][1] == {0: -3, 1: -3, 2: -2}
    assert sel[1][1] == {0: 0, 1: 0}
    assert sel[2][1] == {1: 2}
    assert order == [F[c] for c in "fegh"]
    assert simulate(dag, order)["residency"] == [0, 2, 2, 2, 0]


def _check_incremental(dag):
    s = tree.TreeScheduler(dag)
    checks = [0]

    def on_select(t, gains):
        scratch = s.recompute_gains(set(gains))
        assert scratch == gains
        s.check_tau_delta()
        checks[0] += 1
    order = s.run(on_select)
    s.check_tau_delta()
    assert not check_schedule(dag, order)
    return checks[0]


def test_tree_incremental_gains_equal_from_scratch():
    n = 0
    for seed in range(80):
        dag = Dag(dags.random_dag(seed, n_leaves=int(3 + seed % 6), n_trees=int(2 + seed % 7),
                                  max_ops_per_tree=4, share_p=0.6))
        n += _check_incremental(dag)
    assert n > 300


def test_tree_incremental_gains_typed_dags():
    for seed in range(10):
        dag = Dag(dags.random_dag(seed, n_leaves=8, n_trees=12, typed=True, Lt=2, N=3))
        _check_incremental(dag)
    _check_incremental(Dag(dags.config_c2(N=4, Lt=2, n_loop4=60, n_loop2=4)))
    _check_incremental(Dag(dags.config_c4(N=2, Lt=1, S=2, n_trees=40)))


def test_optimum_bounds_schedulers():
    hit = 0
    for seed in range(120):
        dag = Dag(dags.random_dag(seed, n_leaves=4, n_trees=3, max_ops_per_tree=3, share_p=0.6))
        if len(dag.contractions()) > 9:
            continue
        opt, opt_order = optimum.dp_peak(dag)
        assert simulate(dag, opt_order)["peak"] == opt
        if len(dag.contractions()) <= 7:
            bf, _ = optimum.brute_force_peak(dag)
            assert bf == opt
        ps = simulate(dag, sibling.schedule(dag))["peak"]
        pt = simulate(dag, tree.schedule(dag))["peak"]
        assert ps >= opt and pt >= opt
        hit += pt == opt
    assert hit > 0
    # Table I DAG: optimum 2 = S2
    assert optimum.dp_peak(Dag(dags.fixture_dstar()))[0] == 2
    assert optimum.brute_force_peak(Dag(dags.fixture_dstar()))[0] == 2


def _postorder(dag, r):
    out = []

    def go(u):
        for c in dag.nodes[u].child:
            go(c)
        if dag.nodes[u].child:
            out.append(u)
    go(r)
    return out


def test_single_tree_is_postorder():
    for seed in range(30):
        w = dags.random_dag(seed, n_leaves=10, n_trees=1, max_ops_per_tree=6)
        dag = Dag(w)
        r = dag.trees[0][0]
        # a single tree built without shared operands is a true tree: post-order
        if any(len(n.parents) > 1 for n in dag.nodes.values()):
            continue
        assert tree.schedule(dag) == _postorder(dag, r)          # T-2: left-first post-order
        # sibling: a depth-first post-order with some child order (its first leaf is the
        # lowest id, S-1): every subtree's contractions form a block ending at its root
        order = sibling.schedule(dag)
        pos = {u: i for i, u in enumerate(order)}
        for u in order:
            sub = _postorder(dag, u)
            assert sorted(pos[v] for v in sub) == list(range(pos[u] - len(sub) + 1, pos[u] + 1))


def test_disjoint_trees_do_not_interleave():
    b = dags.Builder("disj", 1, 1, 1)
    roots = []
    for t in range(3):
        l = [b.leaf(dags.LEAF_X, 1) for _ in range(3)]
        x = b.op(dags.OP_X, l[0], l[1], 1)
        roots.append(b.op(dags.OP_X, x, l[2], 1, share=False))
        b.tree(roots[-1])
    dag = Dag(b.w)
    order = sibling.schedule(dag)
    owner = {u: t for t in dag.tree_ids for u in dag.trees[t][1]}
    seq = [owner[u] for u in order]
    assert seq == sorted(seq)


def test_sibling_process_called_once_per_node():
    for seed in range(20):
        dag = Dag(dags.random_dag(seed, n_leaves=8, n_trees=10, share_p=0.7))
        order = sibling.schedule(dag)
        assert sibling.schedule.last_calls == len(dag.nodes)
        assert not check_schedule(dag, order)


@pytest.mark.slow
def test_schedulers_valid_on_configs():
    for w in (dags.config_c1(), dags.config_c2(N=8, Lt=2), dags.config_c3(N=4, Lt=2, S=4),
              dags.config_c4(N=4, Lt=1, S=4, n_trees=200)):
        dag = Dag(w)
        for sch in (sibling.schedule, tree.schedule):
            o = sch(dag)
            assert not check_schedule(dag, o)
