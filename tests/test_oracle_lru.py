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
