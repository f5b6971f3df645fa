"""Pins of the oracle's peer-HBM tier (readings E-10, E-11), independent of
the oracle's own code:

- hand traces on D* (Table I DAG) at cap 3 for the S1 order (derived by hand from
  E-1..E-4 + E-10/E-11, written out in each test's docstring);
- reduction: peer_cap = 0 and no peer leaves give exactly the E-1..E-9 plan (ops and counts);
- closed forms at unbounded peer capacity: every first eviction is a P2P_OUT, every re-fetch
  a P2P_IN, PCIe carries only each leaf's first load and no D2H; with every leaf peer-homed,
  no H2D at all;
- conservation on random DAGs: each P2P_IN of a non-peer-homed tensor follows a P2P_OUT of it
  with no release between; peer bytes in use never exceed peer_cap and return to 0; the
  device-side trace (used, peak, evictions) does not depend on the tier (E-10 changes only
  where a victim's copy goes).
"""
import pytest

from synth import dags
from oracle.dag import Dag
from oracle import lru, tree, sibling

D = dict(zip("abcdefgh", range(8)))
S1 = [D[c] for c in "eghf"]


def _kinds(p):
    return [(k, u) for (k, u) in p["ops"] if k != "FREE"]


def test_dstar_peer_cap1():
    """cap 3, peer_cap 1, S1: before g the LRU victim b (a leaf, host home) has no peer copy and
    the tier is empty -> P2P_OUT b (peer 1/1); before h the victim a finds the tier full ->
    DROP (E-3); f re-fetches a over PCIe (H2D) and b over NVLink (P2P_IN); b's release at f
    frees the tier."""
    p = lru.plan(Dag(dags.fixture_dstar()), S1, 3, peer_cap=1)
    assert _kinds(p) == [("H2D", D["b"]), ("H2D", D["c"]), ("CONTRACT", D["e"]),
                         ("P2P_OUT", D["b"]), ("H2D", D["a"]), ("CONTRACT", D["g"]),
                         ("DROP", D["a"]), ("H2D", D["d"]), ("CONTRACT", D["h"]),
                         ("H2D", D["a"]), ("P2P_IN", D["b"]), ("CONTRACT", D["f"])]
    assert (p["evictions"], p["h2d_count"], p["d2h_count"]) == (2, 5, 0)
    assert (p["p2p_out_count"], p["p2p_in_count"], p["peer_peak_bytes"]) == (1, 1, 1)


def test_dstar_peer_cap2():
    """peer_cap 2: both victims are stashed; only the four first loads cross PCIe."""
    p = lru.plan(Dag(dags.fixture_dstar()), S1, 3, peer_cap=2)
    assert _kinds(p)[3] == ("P2P_OUT", D["b"]) and _kinds(p)[6] == ("P2P_OUT", D["a"])
    assert _kinds(p)[9:11] == [("P2P_IN", D["a"]), ("P2P_IN", D["b"])]
    assert (p["evictions"], p["h2d_count"], p["p2p_out_count"], p["p2p_in_count"], p["peer_peak_bytes"]) == \
        (2, 4, 2, 2, 2)


def test_dstar_peer_home_leaf():
    """a peer-homed (E-11), no peer tier: a's two fetches (g, f) are P2P_IN, its eviction
    before h a DROP; b, c, d and b's re-fetch stay H2D."""
    p = lru.plan(Dag(dags.fixture_dstar()), S1, 3, peer_leaves={D["a"]})
    assert _kinds(p) == [("H2D", D["b"]), ("H2D", D["c"]), ("CONTRACT", D["e"]),
                         ("DROP", D["b"]), ("P2P_IN", D["a"]), ("CONTRACT", D["g"]),
                         ("DROP", D["a"]), ("H2D", D["d"]), ("CONTRACT", D["h"]),
                         ("P2P_IN", D["a"]), ("H2D", D["b"]), ("CONTRACT", D["f"])]
    assert (p["h2d_count"], p["p2p_in_count"], p["p2p_out_count"], p["peer_peak_bytes"]) == (4, 2, 0, 0)


def _random_cases():
    for seed in range(60):
        dag = Dag(dags.random_dag(seed, n_leaves=6, n_trees=6, share_p=0.6, typed=True))
        for order in (tree.schedule(dag), sibling.schedule(dag)):
            unb = lru.plan(dag, order, None)
            for frac in (0.55, 0.7, 0.85):
                cap = max(int(unb["transient_peak"] * frac), 1)
                try:
                    base = lru.plan(dag, order, cap)
                except lru.InfeasibleError:
                    continue
                yield dag, order, cap, base


def test_zero_peer_tier_is_the_plain_plan():
    for dag, order, cap, base in _random_cases():
        for pol in ("lru", "next_use"):
            b = lru.plan(dag, order, cap, policy=pol)
            p = lru.plan(dag, order, cap, policy=pol, peer_cap=0, peer_leaves=())
            assert p["ops"] == b["ops"]
            assert p["p2p_out_count"] == p["p2p_in_count"] == p["peer_peak_bytes"] == 0


def test_unbounded_peer_tier_closed_form():
    """peer_cap = infinity: H2D = one first load per leaf, D2H = 0, P2P_IN = base re-fetches
    (base H2D - first loads), P2P_OUT = number of distinct (tensor, residency) episodes that
    end in an eviction while no peer copy exists = distinct evicted tensors."""
    for dag, order, cap, base in _random_cases():
        p = lru.plan(dag, order, cap, peer_cap=1 << 60)
        leaves = {u for u, n in dag.nodes.items() if not n.child}
        used_leaves = {x for u in order for x in dag.nodes[u].child} & leaves
        assert p["h2d_count"] == len(used_leaves)
        assert p["d2h_count"] == 0
        assert p["p2p_in_count"] == base["h2d_count"] - len(used_leaves)
        evicted = {u for (k, u) in base["ops"] if k in ("D2H", "DROP")}
        assert p["p2p_out_count"] == len(evicted)
        assert p["evictions"] == base["evictions"] and p["used"] == base["used"]


def test_all_leaves_peer_homed_no_pcie():
    for dag, order, cap, base in _random_cases():
        leaves = {u for u, n in dag.nodes.items() if not n.child}
        p = lru.plan(dag, order, cap, peer_cap=1 << 60, peer_leaves=leaves)
        assert p["h2d_count"] == 0 and p["d2h_count"] == 0
        # every leaf fetch of the base plan is now a P2P_IN; intermediates' re-fetches too
        assert p["p2p_in_count"] == base["h2d_count"]


@pytest.mark.parametrize("pol", ["lru", "next_use"])
def test_peer_conservation(pol):
    for dag, order, cap, base in _random_cases():
        leaves = sorted(u for u, n in dag.nodes.items() if not n.child)
        for peer_cap in (0, 1, 3, cap // 2, cap):
            for homed in (set(), set(leaves[::3])):
                p = lru.plan(dag, order, cap, policy=pol, peer_cap=peer_cap, peer_leaves=homed)
                b = lru.plan(dag, order, cap, policy=pol)
                assert p["used"] == b["used"] and p["evictions"] == b["evictions"]
                stashed, peer_bytes, peak = set(), 0, 0
                for k, u in p["ops"]:
                    size = dag.nodes[u].size
                    if k == "P2P_OUT":
                        assert u not in stashed and u not in homed
                        stashed.add(u)
                        peer_bytes += size
                        peak = max(peak, peer_bytes)
                        assert peer_bytes <= peer_cap
                    elif k == "P2P_IN":
                        assert u in stashed or u in homed
                    elif k == "H2D":
                        assert u not in stashed and u not in homed
                    elif k == "FREE" and u in stashed:
                        stashed.discard(u)
                        peer_bytes -= size
                assert peer_bytes == 0 and peak == p["peer_peak_bytes"]
                # PCIe + NVLink fetches together are the base plan's fetches
                assert p["h2d_count"] + p["p2p_in_count"] == b["h2d_count"]
