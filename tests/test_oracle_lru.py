"""Pins of oracle O5 (capacity-limited LRU device plan; readings E-1..E-8).

- hand-computed eviction / transfer counts on D* (Table I DAG) per capacity
  (derived by hand from rules E-1..E-4)
- unbounded capacity reproduces the §II-C memory model exactly
- accounting identities: every D2H is matched by a later re-fetch; final residency 0
- monotonicity in capacity for uniform sizes (LRU stack property)
"""
import numpy as np
import pytest

from synth import dags
from oracle.dag import Dag
from oracle.memory import simulate
from oracle import lru, sibling, tree

D = dict(zip("abcdefgh", range(8)))
S1 = [D[c] for c in "eghf"]
S2 = [D[c] for c in "fegh"]


@pytest.mark.parametrize("cap,s1,s2", [(3, (2, 6), (1, 5)), (4, (1, 5), (0, 4)),
                                        (5, (0, 4), (0, 4)), (100, (0, 4), (0, 4))])
def test_dstar_capacity_table(cap, s1, s2):
    dag = Dag(dags.fixture_dstar())
    for order, (ev, h2d) in ((S1, s1), (S2, s2)):
        p = lru.plan(dag, order, cap)
        assert (p["evictions"], p["h2d_count"]) == (ev, h2d)
        assert p["d2h_count"] == 0          # every victim here is a leaf (E-3)


def test_dstar_cap2_infeasible():
    dag = Dag(dags.fixture_dstar())
    for order in (S1, S2):
        with pytest.raises(lru.InfeasibleError):
            lru.plan(dag, order, 2)


def test_dstar_cap3_S1_trace():
    """Hand trace of S1 at cap 3: e loads b,c (3); g must evict c?  c is dead after e and
    released; before g: used {b,e}=2, need a + g = 2 -> evict LRU non-operand b;
    before h: used {a,e}=2 (g released), need d + h = 2 -> evict a; f re-fetches a and b."""
    dag = Dag(dags.fixture_dstar())
    p = lru.plan(dag, S1, 3)
    kinds = [(k, u) for (k, u) in p["ops"] if k != "FREE"]
    assert kinds == [("H2D", D["b"]), ("H2D", D["c"]), ("CONTRACT", D["e"]),
                     ("DROP", D["b"]), ("H2D", D["a"]), ("CONTRACT", D["g"]),
                     ("DROP", D["a"]), ("H2D", D["d"]), ("CONTRACT", D["h"]),
                     ("H2D", D["a"]), ("H2D", D["b"]), ("CONTRACT", D["f"])]


def _orders(dag):
    yield sibling.schedule(dag)
    yield tree.schedule(dag)


def test_unbounded_equals_memory_model():
    for seed in range(40):
        dag = Dag(dags.random_dag(seed, n_leaves=6, n_trees=6, share_p=0.6))
        for order in _orders(dag):
            sim = simulate(dag, order)
            p = lru.plan(dag, order, None)
            assert p["used"] == sim["residency"]
            assert p["peak"] == sim["peak"] and p["transient_peak"] == sim["transient_peak"]
            assert p["evictions"] == 0 and p["d2h_count"] == 0
            leaves = [u for u in dag.nodes if not dag.nodes[u].child]
            assert p["h2d_count"] == len(leaves)
            assert p["h2d_bytes"] == sum(dag.nodes[u].size for u in leaves)
            # a capacity equal to the transient peak never evicts
            assert lru.plan(dag, order, sim["transient_peak"])["evictions"] == 0


def test_accounting_identities_under_pressure():
    for seed in range(60):
        dag = Dag(dags.random_dag(seed, n_leaves=6, n_trees=8, share_p=0.7, max_size=5))
        for order in _orders(dag):
            sim = simulate(dag, order)
            lo = max(sum(dag.nodes[c].size for c in dag.nodes[u].child) + dag.nodes[u].size
                     for u in order)
            for cap in range(lo, sim["transient_peak"] + 1):
                p = lru.plan(dag, order, cap)
                assert p["peak"] <= cap and p["transient_peak"] <= cap
                # each D2H'd tensor is fetched back at least once later
                d2h = [u for (k, u) in p["ops"] if k == "D2H"]
                for u in d2h:
                    i = p["ops"].index(("D2H", u))
                    assert ("H2D", u) in p["ops"][i:]
                assert len(set(d2h)) == len(d2h)        # E-4: write-once host copy
                assert p["evictions"] == sum(1 for (k, _) in p["ops"] if k in ("D2H", "DROP"))
                n_h2d = sum(1 for (k, _) in p["ops"] if k == "H2D")
                assert n_h2d == p["h2d_count"]


def test_monotone_in_capacity_uniform_sizes():
    for seed in range(40):
        dag = Dag(dags.random_dag(seed, n_leaves=6, n_trees=8, share_p=0.7, max_size=1))
        for order in _orders(dag):
            sim = simulate(dag, order)
            lo = max(len(dag.nodes[u].child) + 1 for u in order)
            ev = [lru.plan(dag, order, c)["evictions"] for c in range(lo, sim["transient_peak"] + 2)]
            assert all(a >= b for a, b in zip(ev, ev[1:]))
            assert ev[-1] == 0


# ---- E-9: next-use (Belady) eviction ---------------------------------------------------------

NU_ORDER = [4, 5, 6, 7, 8]


def test_next_use_hand_trace():
    """fixture_next_use at cap 4 (three unit leaves + the output).  Before s3=(d,b) the
    non-operands a and c are resident: LRU evicts c (touched at s2 before a), which s4
    needs next, and then a for s4, which s5 re-fetches: 2 evictions, 6 H2D.  Next use evicts
    a (read again at s5, after c's read at s4): 1 eviction, 5 H2D (hand-derived)."""
    dag = Dag(dags.fixture_next_use())
    p = lru.plan(dag, NU_ORDER, 4)
    assert (p["evictions"], p["h2d_count"]) == (2, 6)
    q = lru.plan(dag, NU_ORDER, 4, policy="next_use")
    assert (q["evictions"], q["h2d_count"]) == (1, 5)
    kinds = [(k, u) for (k, u) in q["ops"] if k not in ("FREE",)]
    assert kinds == [("H2D", 0), ("H2D", 1), ("CONTRACT", 4), ("H2D", 2), ("CONTRACT", 5),
                     ("DROP", 0), ("H2D", 3), ("CONTRACT", 6), ("CONTRACT", 7),
                     ("H2D", 0), ("CONTRACT", 8)]
    for cap in (5, 100):
        assert lru.plan(dag, NU_ORDER, cap, policy="next_use")["h2d_count"] == 4


def _min_fetches(dag, order, cap):
    """Brute force over every victim choice (E-1 mechanics, any resident non-operand may be
    evicted): the minimum number of H2D fetches.  For root-only DAGs (only leaves are ever
    resident between steps, unit sizes) this is the paging problem whose optimum Belady's
    farthest-next-use rule attains."""
    nodes = dag.nodes
    best = [None]

    def rec(i, resident, fetches):
        if best[0] is not None and fetches >= best[0]:
            return
        if i == len(order):
            best[0] = fetches
            return
        u = order[i]
        ops = nodes[u].child
        need = sum(1 for x in ops if x not in resident) + 1
        if len(resident) + need > cap:
            for v in sorted(resident - set(ops)):
                rec(i, resident - {v}, fetches)
            return
        new = set(resident) | set(ops)
        f = fetches + sum(1 for x in ops if x not in resident)
        # leaves with no later reader are released (E-8)
        later = set(x for w in order[i + 1:] for x in nodes[w].child)
        rec(i + 1, frozenset(x for x in new if x in later), f)

    rec(0, frozenset(), 0)
    return best[0]


def test_next_use_optimal_on_root_only_dags():
    """Belady's theorem as a pin: on random root-only DAGs with unit sizes the next-use plan
    fetches the minimum possible number of leaves (brute force over all victim choices), and
    LRU never beats it."""
    rng = np.random.default_rng(7)
    checked = 0
    for trial in range(120):
        k = int(rng.integers(4, 7))
        m = int(rng.integers(5, 10))
        w = dags.Workload("ro%d" % trial, 1, 1, 1)
        pairs = [tuple(int(x) for x in rng.choice(k, size=2, replace=False)) for _ in range(m)]
        if len(set(x for pr in pairs for x in pr)) < k:
            continue                       # every leaf must be read (no isolated nodes)
        for i in range(k):
            w.nodes.append((i, dags.LEAF_X, -1, -1, 1))
        for j, (a, b) in enumerate(pairs):
            w.nodes.append((k + j, dags.OP_X, a, b, 1))
            w.trees.append((j, k + j))
            w.terms.append((0, j, 1.0, 0.0))
        dag = Dag(w)
        order = [k + j for j in range(m)]
        for cap in range(3, k + 2):
            q = lru.plan(dag, order, cap, policy="next_use")
            p = lru.plan(dag, order, cap)
            opt = _min_fetches(dag, order, cap)
            assert q["h2d_count"] == opt, (trial, cap)
            assert p["h2d_count"] >= opt
            checked += 1
    assert checked > 80


def test_next_use_accounting_on_random_dags():
    """With intermediates (D2H on first eviction, E-4) the next-use plan keeps every E
    accounting identity: final residency 0, every D2H re-fetched, unbounded == LRU."""
    for seed in range(30):
        dag = Dag(dags.random_dag(seed, n_leaves=6, n_trees=6, share_p=0.6))
        order = tree.schedule(dag)
        tp = lru.plan(dag, order)["transient_peak"]
        assert lru.plan(dag, order, None, policy="next_use")["ops"] == lru.plan(dag, order)["ops"]
        for cap in (tp, max(1, tp - 2), max(1, tp // 2)):
            try:
                q = lru.plan(dag, order, cap, policy="next_use")
            except lru.InfeasibleError:
                continue
            h2d_inter = sum(1 for (kk, u) in q["ops"] if kk == "H2D" and dag.nodes[u].child)
            assert h2d_inter >= q["d2h_count"]
