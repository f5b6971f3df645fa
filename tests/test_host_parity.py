"""Bit-exact parity of the C++ host library (libcc.so, host-only context) with the oracle.

Integers only (CPU): schedule order (sibling Alg. 1-3, tree Alg. 4-8), tree selection
order, §II-C memory trace (M_i and transients), LRU plan op queue and counters
(evictions, transfers, bytes, peaks), partitions, validation error classes.
"""
import os
import re
import subprocess

import pytest

from synth import dags
from oracle.dag import Dag, OracleError
from oracle import sibling, tree, lru, partition
from oracle.memory import simulate

cc = pytest.importorskip("paper_2511_02257_b200.cc")


def _ctx(w):
    c = cc.Context(-1)
    c.load_workload(w)
    return c


def _check(w, caps=(None,)):
    dag = Dag(w)
    c = _ctx(w)
    s_or = sibling.schedule(dag)
    s_cc, st = c.schedule(cc.CC_SIBLING)
    assert s_cc == s_or
    sim = simulate(dag, s_or)
    m, tr = c.memory_trace()
    assert m == sim["residency"] and tr == sim["transient"]
    assert st["model_peak"] == sim["peak"] and st["model_transient_peak"] == sim["transient_peak"]
    ts = tree.TreeScheduler(dag)
    t_or = ts.run()
    t_cc, _ = c.schedule(cc.CC_TREE)
    assert t_cc == t_or
    assert c.tree_order() == ts.tree_order
    for order, algo in ((s_or, cc.CC_SIBLING), (t_or, cc.CC_TREE)):
        for cap in caps:
            try:
                p = lru.plan(dag, order, cap)
            except lru.InfeasibleError:
                with pytest.raises(cc.CCError) as ei:
                    c.schedule(algo, cap_bytes=cap or 0)
                assert ei.value.code == "INFEASIBLE"
                continue
            _, st = c.schedule(algo, cap_bytes=cap or 0)
            for k in ("evictions", "h2d_count", "d2h_count", "h2d_bytes", "d2h_bytes", "peak",
                      "transient_peak"):
                assert st[k] == p[k], (k, cap)
            assert st["host_peak_bytes"] == p["host_peak_bytes"]
            ops = [(k, n) for (k, n, _, _) in c.plan_ops()]
            assert ops == p["ops"]
        # the GIVEN path replays an arbitrary valid order
        _, st = c.schedule(cc.CC_GIVEN, given=order)
        assert st["model_peak"] == simulate(dag, order)["peak"]
    return dag


def test_fixtures_exact():
    _check(dags.fixture_dstar(), caps=(None, 2, 3, 4, 5))
    _check(dags.fixture_f1(), caps=(None, 2, 3, 4, 5))


def test_random_abstract_dags():
    for seed in range(250):
        w = dags.random_dag(seed, n_leaves=3 + seed % 7, n_trees=1 + seed % 9,
                            max_ops_per_tree=1 + seed % 5, share_p=(seed % 10) / 10, max_size=1 + seed % 6)
        dag = Dag(w)
        tp = simulate(dag, sibling.schedule(dag))["transient_peak"]
        _check(w, caps=(None, tp, max(1, tp - 2), max(1, tp // 2)))


def test_random_typed_dags():
    for seed in range(30):
        w = dags.random_dag(seed, n_leaves=8, n_trees=15, typed=True, Lt=3, N=5)
        _check(w, caps=(None, 16 * 3 * 25 * 4, 16 * 3 * 25 * 6))


def test_configs_small_scale():
    mes = 16 * 2 * 8 * 8
    _check(dags.config_c1(), caps=(None,))
    _check(dags.config_c2(N=8, Lt=2), caps=(None, 6 * mes, 10 * mes))
    _check(dags.config_c3(N=4, Lt=2, S=4), caps=(None,))
    _check(dags.config_c4(N=4, Lt=1, S=4, n_trees=300), caps=(None, 16 * 4 * 64 * 6, 16 * 4 * 64 * 9))
    # tritium-like BxBxB (f4): baryon 16 Lt S N^3, tetra 16 Lt N^4, meson 16 Lt N^2 mixed
    bary = 16 * 2 * 4 * 4 ** 3
    _check(dags.config_c6(N=4, Lt=2, S=4, n_trees=150), caps=(None, 5 * bary, 8 * bary))


def test_c6_sizes_flops_and_text_roundtrip(tmp_path):
    """BxBxB node sizes / dag stats agree with the oracle, the text format knows the new kinds,
    and a contract-all kind used as an interior node (or a GEMM kind as a root) is rejected."""
    w = dags.config_c6(N=5, Lt=3, S=2, n_trees=40)
    dag = Dag(w)
    c = _ctx(w)
    assert c.dag_info()["V"] == len(dag.nodes)
    _, st = c.schedule(cc.CC_TREE)
    assert st["model_peak"] == simulate(dag, tree.schedule(dag))["peak"]
    p = tmp_path / "c6.txt"
    p.write_text(w.to_text())
    c2 = cc.Context(-1)
    c2.load_dag_file(str(p))
    assert c2.schedule(cc.CC_TREE)[0] == c.schedule(cc.CC_TREE)[0]
    b = dags.Builder("bad", 1, 2, 2)
    x, y = b.leaf(dags.LEAF_B), b.leaf(dags.LEAF_B)
    r = b.op(dags.BB3, x, y)
    b.tree(b.op(dags.BB3, r, y))
    for w_bad in (b.w,):
        with pytest.raises(OracleError):
            Dag(w_bad)
        with pytest.raises(cc.CCError) as ei:
            _ctx(w_bad)
        assert ei.value.code == "INCONSISTENT"


@pytest.mark.slow
def test_configs_full_scale_integers():
    _check(dags.config_c2(), caps=(None, 1 << 30))
    _check(dags.config_c4(), caps=(None, 32 * 10 ** 9))


def test_dag_stats_match():
    for w in (dags.fixture_dstar(), dags.config_c2(N=8, Lt=2), dags.config_c4(N=4, Lt=1, S=4, n_trees=100)):
        s_or = Dag(w).stats()
        s_cc = _ctx(w).dag_info()
        for k in ("V", "E", "k", "n_contr", "max_rank"):
            assert s_cc[k] == s_or[k]
        assert s_cc["F_v"] == pytest.approx(s_or["F_v"], rel=1e-15)
        assert s_cc["F_e"] == pytest.approx(s_or["F_e"], rel=1e-15)


def _err(w):
    try:
        Dag(w)
        o = None
    except OracleError as e:
        o = e.code
    try:
        _ctx(w)
        c = None
    except cc.CCError as e:
        c = e.code
    return o, c


def test_validation_error_classes():
    L, O = dags.LEAF_X, dags.OP_X
    base = [(0, L, -1, -1, 1), (1, L, -1, -1, 1)]
    cases = [
        dags.Workload("cyc", 1, 1, 1, nodes=base + [(2, O, 0, 3, 1), (3, O, 2, 1, 1), (4, O, 3, 0, 1)], trees=[(0, 4)]),
        dags.Workload("same", 1, 1, 1, nodes=base + [(2, O, 0, 0, 1)], trees=[(0, 2)]),
        dags.Workload("multi", 1, 1, 1, nodes=base + [(2, O, 0, 1, 1)], trees=[(0, 2), (1, 2)]),
        dags.Workload("unk", 1, 1, 1, nodes=base + [(2, O, 0, 9, 1)], trees=[(0, 2)]),
        dags.Workload("dup", 1, 1, 1, nodes=base + [(1, L, -1, -1, 1)], trees=[]),
        dags.Workload("kind", 2, 2, 2, nodes=[(0, dags.LEAF_M, -1, -1, 0), (1, dags.LEAF_B, -1, -1, 0),
                                              (2, dags.MM1, 0, 1, 0), (3, dags.TR_MM, 2, 0, 0)], trees=[(0, 3)]),
        dags.Workload("noroot", 1, 1, 1, nodes=base + [(2, O, 0, 1, 1)], trees=[]),
        dags.Workload("badterm", 1, 1, 1, nodes=base + [(2, O, 0, 1, 1)], trees=[(0, 2)], terms=[(0, 5, 1.0, 0.0)]),
    ]
    for w in cases:
        o, c = _err(w)
        assert o is not None and o == c, (w.name, o, c)


def test_text_file_load(tmp_path):
    for w in (dags.fixture_dstar(), dags.config_c2(N=8, Lt=2, n_loop4=40)):
        p = tmp_path / (w.name + ".txt")
        p.write_text(w.to_text())
        c = cc.Context(-1)
        c.load_dag_file(str(p))
        assert c.schedule(cc.CC_TREE)[0] == tree.schedule(Dag(w))
    bad = tmp_path / "bad.txt"
    bad.write_text("dims 1 1 1\nnode 0 leafX size 1\nnode 1 bogus 0 0\n")
    with pytest.raises(cc.CCError, match="line 3"):
        cc.Context(-1).load_dag_file(str(bad))


def test_tree_partitions_match_oracle():
    for w, n in ((dags.config_c2(N=8, Lt=2), 3), (dags.config_c4(N=4, Lt=1, S=4, n_trees=300), 4),
                 (dags.config_c5(N=8, Lt=2, n_pairs=60, n_trees=400), 8)):
        dag = Dag(w)
        parts = partition.tree_parts(dag, n)
        c = _ctx(w)
        seen = set()
        for p in range(n):
            c.partition(n, p, cc.PART_TREES)
            mine = c.part_trees()
            assert mine == sorted(t for t, q in parts.items() if q == p)
            seen |= set(mine)
            sub = partition.sub_workload(w, mine)
            sd = Dag(sub)
            assert c.schedule(cc.CC_TREE)[0] == tree.schedule(sd)
        assert seen == set(dag.tree_ids)


def test_time_partitions_sizes():
    w = dags.config_c2(N=8, Lt=6, n_loop4=30)
    c = _ctx(w)
    for p in range(4):
        c.partition(4, p, cc.PART_TIME)
        t0, t1 = partition.time_range(6, 4, p)
        wp = dags.Workload(w.name, t1 - t0, w.N, w.S, nodes=w.nodes, trees=w.trees, terms=w.terms)
        dag = Dag(wp)
        order, st = c.schedule(cc.CC_TREE)
        assert order == tree.schedule(dag)
        assert st["peak"] == simulate(dag, order)["peak"]


def test_abi_exports_every_declared_symbol(repo_root):
    hdr = open(os.path.join(repo_root, "include", "cc.h")).read()
    declared = set(re.findall(r"^\s*(?:cc_status|void|const char\*|size_t)\s+(cc_\w+)\s*\(", hdr, re.M))
    out = subprocess.run(["nm", "-D", "--defined-only", cc.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cc_\w+)$", out, re.M))
    assert declared and declared <= exported, declared - exported
    assert set(cc.EXPORTED) == declared


def test_device_calls_fail_on_host_only_ctx():
    c = _ctx(dags.config_c1())
    c.schedule(cc.CC_TREE)
    with pytest.raises(cc.CCError) as e:
        c.execute()
    assert e.value.code == "STATE"


def test_rsgs_matches_oracle():
    """CC_RSGS (RS-GS-like baseline, readings R-1..R-4) == oracle/rsgs.py, order and chain,
    on random DAGs and the configs at full scale; plans under caps too."""
    from oracle import rsgs
    cases = [dags.fixture_dstar(), dags.fixture_f1()]
    cases += [dags.random_dag(s, n_leaves=3 + s % 7, n_trees=1 + s % 9, max_ops_per_tree=1 + s % 5,
                              share_p=(s % 10) / 10, max_size=1 + s % 6) for s in range(120)]
    cases += [dags.config_c2(), dags.config_c4(), dags.config_c5(N=256, n_pairs=400, n_trees=3000)]
    for w in cases:
        dag = Dag(w)
        c = _ctx(w)
        o_cc, st = c.schedule(cc.CC_RSGS)
        assert o_cc == rsgs.schedule(dag)
        assert c.tree_order() == rsgs.tree_chain(dag)
        sim = simulate(dag, o_cc)
        assert st["model_peak"] == sim["peak"]
    w = dags.config_c4(N=8, Lt=1, S=4, n_trees=200)
    dag = Dag(w)
    order = rsgs.schedule(dag)
    c = _ctx(w)
    for cap in (None, 12 * 16 * 4 * 8 ** 3, 7 * 16 * 4 * 8 ** 3):
        p = lru.plan(dag, order, cap)
        _, st = c.schedule(cc.CC_RSGS, cap_bytes=cap or 0)
        for k in ("evictions", "h2d_count", "d2h_count", "h2d_bytes", "d2h_bytes", "peak", "transient_peak"):
            assert st[k] == p[k], (k, cap)


def _check_next_use(w, caps):
    """C++ next-use (E-9) plans == oracle plans: counters, bytes, peaks and the op queue."""
    dag = Dag(w)
    c = _ctx(w)
    for algo, order in ((cc.CC_TREE, tree.schedule(dag)), (cc.CC_SIBLING, sibling.schedule(dag))):
        for cap in caps:
            try:
                p = lru.plan(dag, order, cap, policy="next_use")
            except lru.InfeasibleError:
                with pytest.raises(cc.CCError):
                    c.schedule(algo, cap_bytes=cap or 0, evict_next_use=True)
                continue
            _, st = c.schedule(algo, cap_bytes=cap or 0, evict_next_use=True)
            for k in ("evictions", "h2d_count", "d2h_count", "h2d_bytes", "d2h_bytes", "peak",
                      "transient_peak", "host_peak_bytes"):
                assert st[k] == p[k], (k, cap)
            assert [(k, n) for (k, n, _, _) in c.plan_ops()] == p["ops"]


def test_next_use_plans_bit_exact():
    w = dags.fixture_next_use()
    dag = Dag(w)
    c = _ctx(w)
    _, st = c.schedule(cc.CC_GIVEN, given=[4, 5, 6, 7, 8], cap_bytes=4, evict_next_use=True)
    assert (st["evictions"], st["h2d_count"]) == (1, 5)
    assert [(k, n) for (k, n, _, _) in c.plan_ops()] == lru.plan(dag, [4, 5, 6, 7, 8], 4, policy="next_use")["ops"]
    _check_next_use(dags.fixture_dstar(), caps=(None, 2, 3, 4, 5))
    for seed in range(60):
        w = dags.random_dag(seed, n_leaves=7, n_trees=7, share_p=0.6)
        tp = lru.plan(Dag(w), tree.schedule(Dag(w)))["transient_peak"]
        _check_next_use(w, caps=(None, tp, max(1, tp - 2), max(1, tp // 2)))
    mes = 16 * 2 * 8 * 8
    _check_next_use(dags.config_c2(N=8, Lt=2), caps=(6 * mes, 10 * mes))
    _check_next_use(dags.config_c4(N=4, Lt=1, S=4, n_trees=300), caps=(16 * 4 * 64 * 6, 16 * 4 * 64 * 9))


def test_next_use_c4_full_scale():
    """c4 at full scale under its 32e9 B cap: bit-exact with the oracle, and fewer bytes over
    PCIe than LRU (the point of E-9)."""
    w = dags.config_c4()
    _check_next_use(w, caps=(32 * 10 ** 9,))
    c = _ctx(w)
    _, lru_st = c.schedule(cc.CC_TREE, cap_bytes=32 * 10 ** 9)
    _, nu_st = c.schedule(cc.CC_TREE, cap_bytes=32 * 10 ** 9, evict_next_use=True)
    assert nu_st["h2d_bytes"] + nu_st["d2h_bytes"] < lru_st["h2d_bytes"] + lru_st["d2h_bytes"]


def test_ozaki_workspace_sizes_host_only():
    """The Ozaki engine's workspace queries are host functions (no GPU): 0 for invalid
    arguments, the full-batch size grows with Lt and with the slice count, BB2's K chunks add
    split-K partials, MM1 via the generic query equals the MM1-specific one."""
    assert cc.cc_mm1_ozaki_workspace_bytes(0, 128, 5) == 0
    assert cc.cc_mm1_ozaki_workspace_bytes(4, 128, 3) == 0
    assert cc.cc_gemm_ozaki_workspace_bytes(cc.CC_TR_MM, 4, 128, 1, 5) == 0
    a = cc.cc_gemm_ozaki_workspace_bytes(cc.CC_MM1, 4, 128, 1, 5)
    assert a == cc.cc_mm1_ozaki_workspace_bytes(4, 128, 5) > 0
    assert cc.cc_gemm_ozaki_workspace_bytes(cc.CC_MM1, 8, 128, 1, 5) > a
    assert cc.cc_gemm_ozaki_workspace_bytes(cc.CC_MM1, 4, 128, 1, 6) > a
    # BB2 N=16 S=64: K = 16384 complex -> Kp = 32768 bytes -> 2 chunks of 16 KB (partials)
    one = cc.cc_gemm_ozaki_workspace_bytes(cc.CC_BB2, 1, 16, 64, 5)
    slices = 5 * 128 * 32768 + 5 * 64 * 32768           # A slices (Mp=128) + B slices (2*32 rows)
    assert one >= slices + 2 * 128 * 32 * 16            # + 2 chunks of [Mp][Nc] complex partials


PEER_KEYS = ("evictions", "h2d_count", "d2h_count", "h2d_bytes", "d2h_bytes", "peak", "transient_peak",
             "host_peak_bytes", "p2p_out_count", "p2p_out_bytes", "p2p_in_count", "p2p_in_bytes", "peer_peak_bytes")


def _check_peer(w, cap, peer_caps, homed_sets, algo=None):
    dag = Dag(w)
    c = _ctx(w)
    order, _ = c.schedule(cc.CC_TREE if algo is None else algo)
    for pol, nu in (("lru", False), ("next_use", True)):
        for pc in peer_caps:
            for homed in homed_sets:
                try:
                    p = lru.plan(dag, order, cap, policy=pol, peer_cap=pc, peer_leaves=homed)
                except lru.InfeasibleError:
                    continue
                _, st = c.schedule(cc.CC_GIVEN, given=order, cap_bytes=cap or 0, evict_next_use=nu,
                                   peer_cap_bytes=pc, peer_leaves=homed)
                for k in PEER_KEYS:
                    assert st[k] == p[k], (k, pol, pc)
                assert [(k, n) for (k, n, _, _) in c.plan_ops()] == p["ops"]


def test_peer_tier_plans_bit_exact():
    """Peer-HBM tier (readings E-10, E-11): the C++ plan's op queue and counters equal the
    oracle's on D*, random typed DAGs and small c2/c4 shapes, for LRU and next-use eviction."""
    D = dict(zip("abcdefgh", range(8)))
    _check_peer(dags.fixture_dstar(), 3, (0, 1, 2, 10), (set(), {D["a"]}, {D["a"], D["b"], D["d"]}))
    for seed in range(40):
        w = dags.random_dag(seed, n_leaves=7, n_trees=7, share_p=0.6, typed=True)
        dag = Dag(w)
        tp = lru.plan(dag, tree.schedule(dag))["transient_peak"]
        leaves = sorted(u for u, n in dag.nodes.items() if not n.child)
        for cap in (max(1, tp * 2 // 3), max(1, tp // 2)):
            _check_peer(w, cap, (0, cap // 3, cap, 1 << 50), (set(), set(leaves[::2])))
    w = dags.config_c4(N=4, Lt=1, S=4, n_trees=300)
    baryon = 16 * 4 * 64
    leaves = sorted(n[0] for n in w.nodes if n[1] in (dags.LEAF_M, dags.LEAF_B))
    _check_peer(w, 9 * baryon, (0, 3 * baryon, 40 * baryon), (set(), set(leaves[:4])))


def test_peer_tier_c4_full_scale():
    """c4 at full scale (32e9 B cap) with a 32e9 B peer tier: bit-exact with the oracle, and the
    PCIe bytes fall below the plain plan's (the point of E-10)."""
    w = dags.config_c4()
    _check_peer(w, 32 * 10 ** 9, (32 * 10 ** 9,), (set(),))
    c = _ctx(w)
    _, base = c.schedule(cc.CC_TREE, cap_bytes=32 * 10 ** 9, evict_next_use=True)
    _, peer = c.schedule(cc.CC_TREE, cap_bytes=32 * 10 ** 9, evict_next_use=True, peer_cap_bytes=32 * 10 ** 9)
    assert peer["h2d_bytes"] + peer["d2h_bytes"] < base["h2d_bytes"] + base["d2h_bytes"]
    assert peer["h2d_count"] + peer["p2p_in_count"] == base["h2d_count"]


def test_grid_partition_part_info_leaf_owners():
    """GRID split (M-2), replication (M-3) and leaf owners (E-11): the C++ part's trees, time
    range, work / replication counters and leaf owners equal the oracle's, and each part's
    plan is bit-exact with the oracle on that part's sub-workload."""
    cases = [(dags.config_c5(N=8, Lt=8, n_pairs=40, n_trees=200), 2, 2),
             (dags.config_c5(N=8, Lt=8, n_pairs=40, n_trees=200), 3, 4),
             (dags.config_c4(N=4, Lt=2, S=4, n_trees=120), 2, 2),
             (dags.config_c6(N=4, Lt=2, S=4, n_trees=40), 2, 2),
             (dags.fixture_dstar(), 2, 1)]
    for w, nT, nL in cases:
        dag = Dag(w)
        parts = partition.tree_parts(dag, nT)
        owners = partition.leaf_owners(w, nT)
        for p in range(nT * nL):
            c = _ctx(w)
            c.partition_grid(nT, nL, p)
            pt, ptm = partition.grid_part(nT, nL, p)
            assert c.part_trees() == sorted(t for t in dag.tree_ids if parts[t] == pt)
            if w.Lt > 1 or nL == 1:
                assert c.part_time_range() == partition.time_range(w.Lt, nL, ptm)
            assert c.part_info() == partition.part_stats(w, nT, p, n_time=nL)
            assert c.leaf_owners() == owners
            sub = partition.sub_workload(w, c.part_trees())
            t0, t1 = partition.time_range(w.Lt, nL, ptm)
            sub.Lt = t1 - t0
            sd = Dag(sub)
            order, st = c.schedule(cc.CC_TREE)
            assert order == tree.schedule(sd)
            assert st["peak"] == lru.plan(sd, order)["peak"]
    c = _ctx(dags.config_c5(N=8, Lt=8, n_pairs=40, n_trees=200))
    assert c.part_info()["replicated_work"] == 0
    with pytest.raises(cc.CCError):
        c.leaf_owners()


def _check_placement(c, w, pool):
    """Replays cc_phys_ops: every allocation, move destination and contraction output lands
    inside the pool on bytes no live tensor holds, moves read a live tensor at its current
    offset, and contractions read their operands where the plan last put them."""
    dag = Dag(w)
    size = {u: n.size for u, n in dag.nodes.items()}
    rb = lambda u: (size[u] + 1023) // 1024 * 1024   # noqa: E731
    live = {}

    def free_at(off, b, ignore=None):
        return all(o + rb(u) <= off or off + b <= o for u, o in live.items() if u != ignore)

    moves = 0
    for (kind, node, nbytes, off, dst, off_a, off_b) in c.phys_ops():
        name = cc.OP_KINDS[kind] if kind < len(cc.OP_KINDS) else "MOVE"
        if name == "MOVE":
            assert live.get(node) == off and 0 <= dst and dst + rb(node) <= pool
            assert free_at(dst, rb(node), ignore=node) and (dst + rb(node) <= off or off + rb(node) <= dst)
            live[node] = dst
            moves += 1
        elif name in ("H2D", "P2P_IN"):
            assert 0 <= off and off + rb(node) <= pool and free_at(off, rb(node))
            live[node] = off
        elif name == "CONTRACT":
            n = dag.nodes[node]
            assert off_a == live[n.child[0]] and off_b == live[n.child[1]]
            if off >= 0:
                assert off + rb(node) <= pool and free_at(off, rb(node))
                live[node] = off
        elif name in ("D2H", "P2P_OUT", "DROP", "FREE"):
            live.pop(node, None)
    return moves


def test_compaction_placement_invariants():
    """Physical-pool compaction: where best fit fails for fragmentation, the compacting
    placement succeeds with a few device-to-device moves, and the replayed placement is sound
    (`_check_placement`); with room to spare it makes no moves."""
    hits = 0
    for seed in range(12):
        w = dags.config_c4(N=8, Lt=1, S=4, n_snk=4, n_src=4, n_mes=4, n_trees=40, seed=seed)
        c = _ctx(w)
        baryon = 16 * 4 * 8 ** 3
        for capk in (6, 8):
            try:
                _, st = c.schedule(cc.CC_TREE, cap_bytes=capk * baryon)
            except cc.CCError:
                continue
            tp = st["transient_peak"]
            for pool in range((tp + 1023) // 1024 * 1024, tp * 5 // 4, 1024):
                try:
                    c.phys_plan(pool)
                    assert _check_placement(c, w, pool) == 0
                    continue
                except cc.CCError as e:
                    assert e.code == "NOMEM"
                try:
                    s2 = c.phys_plan(pool, compact=True)
                except cc.CCError:
                    continue
                assert s2["n_moves"] > 0 and _check_placement(c, w, pool) == s2["n_moves"]
                hits += 1
            assert c.phys_plan(tp * 4, compact=True)["n_moves"] == 0     # room to spare: no moves
    assert hits > 0
