"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Tolerance (north_star): complex-FP64 values within 1e-10 relative.  With
phase-limited leaves (synth.rng mode 0) every product in a contraction has phase within
+-19 deg, so |sum| >= 0.94 sum|terms| and an element-wise relative test is meaningful;
random-phase data is checked against the error scale |A|@|B| instead (reading V-4).
Integers (schedules, plans) are bit-exact and covered on CPU in test_host_parity.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import dags, rng as srng  # noqa: E402
from oracle import values, lru, tree, partition  # noqa: E402
from oracle.dag import Dag  # noqa: E402
from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close, device_from, to_numpy_c  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_02257_b200 import cc
    return cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))


def _phase_limited(shape, seed, sigma=1.0):
    n = int(np.prod(shape))
    return srng.leaf_values(seed, 1000 + seed, 0, n, sigma).reshape(shape)


def _random_phase(shape, seed):
    n = int(np.prod(shape))
    return srng.leaf_values(seed, 2000 + seed, 0, n, 1.0, srng.MODE_RANDOM_PHASE).reshape(shape)


def _rel_check(got, want, rel=1e-10):
    err = np.abs(got - want) / np.abs(want)
    assert float(err.max()) <= rel, float(err.max())


def test_fill_synthetic_bit_exact(ctx):
    for (leaf, e0, n, sigma, mode) in ((3, 0, 4096, 1 / 64, 0), (7, 123457, 1000, srng.baryon_sigma(16, 64), 0),
                                       (11, 5, 333, 0.5, 1)):
        d = torch.empty(2 * n, dtype=torch.float64, device="cuda")
        ctx.fill_synthetic(d, n, 42, leaf, e0, mode, sigma)
        torch.cuda.synchronize()
        got = d.cpu().numpy().view(np.complex128)
        want = srng.leaf_values(42, leaf, e0, n, sigma, mode)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("Lt,N", [(1, 8), (2, 33), (3, 64), (2, 100), (4, 128), (1, 200), (2, 256)])
def test_mm1_elementwise(ctx, Lt, N):
    A = _phase_limited((Lt, N, N), 1, 1 / N)
    B = _phase_limited((Lt, N, N), 2, 1 / N)
    C = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
    ctx.mm1(dA := device_from(A), dB := device_from(B), C, Lt, N)
    torch.cuda.synchronize()
    _rel_check(to_numpy_c(C, (Lt, N, N)), values.mm1(A, B))


def test_mm1_random_phase_and_closed_forms(ctx):
    Lt, N = 3, 96
    A = _random_phase((Lt, N, N), 3)
    B = _random_phase((Lt, N, N), 4)
    C = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
    ctx.mm1(dA := device_from(A), dB := device_from(B), C, Lt, N)
    torch.cuda.synchronize()
    got = to_numpy_c(C, (Lt, N, N))
    scale = np.matmul(np.abs(A), np.abs(B))
    assert np.all(np.abs(got - values.mm1(A, B)) <= 1e-13 * scale)
    # all-ones: MM1(J, J) = N J exactly; identity: MM1(I, X) = X exactly
    J = np.ones((Lt, N, N), complex)
    ctx.mm1(dJ := device_from(J), dJ, C, Lt, N)
    torch.cuda.synchronize()
    assert np.array_equal(to_numpy_c(C, (Lt, N, N)), N * J)
    I = np.broadcast_to(np.eye(N, dtype=complex), (Lt, N, N)).copy()
    ctx.mm1(dI := device_from(I), dA, C, Lt, N)
    torch.cuda.synchronize()
    assert np.array_equal(to_numpy_c(C, (Lt, N, N)), A)


@pytest.mark.parametrize("Lt,N,S", [(2, 8, 4), (1, 12, 64), (2, 16, 8), (1, 33, 2)])
def test_bm1_elementwise(ctx, Lt, N, S):
    A = _phase_limited((Lt, S, N, N, N), 5, 1 / np.sqrt(S * N ** 3))
    M = _phase_limited((Lt, N, N), 6, 1 / N)
    C = torch.empty(Lt * S * N ** 3 * 2, dtype=torch.float64, device="cuda")
    ctx.bm1(dA := device_from(A), dM := device_from(M), C, Lt, N, S)
    torch.cuda.synchronize()
    _rel_check(to_numpy_c(C, (Lt, S, N, N, N)), values.bm1(A, M))


@pytest.mark.parametrize("Lt,N,S", [(2, 8, 4), (1, 12, 64), (2, 16, 8), (1, 20, 3), (3, 32, 64)])
def test_bb2_elementwise(ctx, Lt, N, S):
    A = _phase_limited((Lt, S, N, N, N), 7, 1 / np.sqrt(S * N ** 3))
    B = _phase_limited((Lt, S, N, N, N), 8, 1 / np.sqrt(S * N ** 3))
    C = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
    ctx.bb2(dA := device_from(A), dB := device_from(B), C, Lt, N, S)
    torch.cuda.synchronize()
    _rel_check(to_numpy_c(C, (Lt, N, N)), values.bb2(A, B))


@pytest.mark.parametrize("Lt,N", [(1, 8), (4, 32), (3, 33), (2, 100), (64, 128), (2, 257)])
def test_tr_mm(ctx, Lt, N):
    A = _phase_limited((Lt, N, N), 9, 1 / N)
    B = _phase_limited((Lt, N, N), 10, 1 / N)
    c = torch.empty(2 * Lt, dtype=torch.float64, device="cuda")
    ctx.tr_mm(dA := device_from(A), dB := device_from(B), c, Lt, N)
    torch.cuda.synchronize()
    _rel_check(to_numpy_c(c, (Lt,)), values.tr_mm(A, B))
    J = np.ones((Lt, N, N), complex)
    ctx.tr_mm(dJ := device_from(J), dJ, c, Lt, N)
    torch.cuda.synchronize()
    assert np.array_equal(to_numpy_c(c, (Lt,)), np.full(Lt, N * N, complex))


# ---- whole DAGs through cc_execute -----------------------------------------------------------

def test_c1_all_ones_exact():
    w = dags.config_c1()
    _, roots, corr, st, ex = run_gpu(w, leaf_fn=lambda u, op: np.ones((w.Lt, w.N, w.N), complex))
    assert np.array_equal(roots[0], np.full(w.Lt, float(w.N) ** 4, complex))     # N^4 = 2^20
    assert ex["n_kernels"] >= 2


def test_c1_synthetic():
    w = dags.config_c1()
    dag = Dag(w)
    _, roots, corr, st, ex = run_gpu(w)
    r_or, c_or = values.run_workload(w, dag)
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)
    assert ex["h2d_bytes"] == 4 * 16 * w.Lt * w.N ** 2


@pytest.mark.parametrize("flags", [0, 1, 2, 16, 17])
def test_c2_small_all_modes(flags):
    """flags 0/1: dataflow workers (stream / CUDA graph); 2: op-by-op with per-kernel
    timing; 16/17: op-by-op launches (stream / graph)."""
    w = dags.config_c2(N=40, Lt=3, n_loop4=80, n_loop2=6, n_corr=4)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    _, roots, corr, st, ex = run_gpu(w, flags=flags)
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)


def test_correlators_bulk_read():
    """cc_correlators (one copy of every correlator) == cc_correlator per id, also on a TIME part."""
    from paper_2511_02257_b200 import cc
    w = dags.config_c2(N=24, Lt=4, n_loop4=30, n_loop2=4, n_corr=5)
    for part in (None, (2, 1, cc.PART_TIME)):
        ctx, roots, corr, st, ex = run_gpu(w, part=part)
        allc = ctx.correlators()
        _, n, ids = ctx.correlator_device_ptr()
        assert allc.shape[0] == n
        for k, c in enumerate(ids):
            assert np.array_equal(allc[k], corr[c])


def test_schedule_and_mode_invariance_bitwise():
    """Deterministic kernels, no atomics in any reduction: root values are bit-identical run to
    run and across graph/stream mode; with trace fusion off also across schedulers and
    host/device leaves (which traces fuse into which GEMM depends on the plan, and a fused
    trace sums in tile order, so with fusion on those agree to rounding)."""
    from paper_2511_02257_b200 import cc
    w = dags.config_c2(N=24, Lt=2, n_loop4=40, n_loop2=4, n_corr=3)
    fz = {"trace_fusion": 1}
    base = run_gpu(w, algo=cc.CC_TREE, options=fz)[1]
    again = run_gpu(w, algo=cc.CC_TREE, options=fz)[1]
    for t in base:
        assert np.array_equal(base[t], again[t])
    for kw in (dict(algo=cc.CC_SIBLING), dict(algo=cc.CC_RSGS), dict(device_leaves=True),
               dict(flags=1, device_leaves=True)):
        assert_roots_close(run_gpu(w, options=fz, **kw)[1], base, rel=1e-13)
    dl = run_gpu(w, device_leaves=True, options=fz)[1]
    dlg = run_gpu(w, flags=1, device_leaves=True, options=fz)[1]
    for t in dl:
        assert np.array_equal(dl[t], dlg[t])
    base = run_gpu(w, algo=cc.CC_TREE)[1]
    for kw in (dict(algo=cc.CC_SIBLING), dict(algo=cc.CC_RSGS), dict(flags=1), dict(device_leaves=True),
               dict(flags=1, device_leaves=True), dict(options={"precopy": 0}), dict(options={"early_copies": 0}),
               dict(options={"copy_reorder": 0, "tr_ratio": 0.5}), dict(options={"slice_major": 0}),
               dict(flags=1, device_leaves=True, options={"slice_major": 0})):
        other = run_gpu(w, **kw)[1]
        for t in base:
            assert np.array_equal(base[t], other[t]), kw
    # the op-by-op path (stream-K kernels) sums in another order: equal within tolerance
    legacy = run_gpu(w, flags=16)[1]
    assert_roots_close(legacy, base, rel=1e-13)


def test_chunked_and_reordered_h2d_copies():
    """Host leaves copied in time-slice chunks (items wait only for the chunk holding their
    slice) and wait-free copies moved ahead in queue order: same values as the oracle and
    bit-identical to whole-tensor copies in plan order (the copy schedule never changes
    the arithmetic)."""
    w = dags.config_c2(N=40, Lt=8, n_loop4=60, n_loop2=6, n_corr=4)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    base = run_gpu(w, options={"h2d_chunk_bytes": 100 << 20, "copy_reorder": 0})[1]
    for chunk, reorder in ((65536, 0), (65536, 1), (10 << 10, 1), (100 << 20, 1)):
        opt = {"h2d_chunk_bytes": chunk, "copy_reorder": reorder}
        for flags in (0, 1):
            _, roots, corr, st, ex = run_gpu(w, flags=flags, options=opt)
            assert_roots_close(roots, r_or)
            assert_corr_close(dag, r_or, corr, c_or)
            for t in base:
                assert np.array_equal(base[t], roots[t]), (chunk, reorder, flags)
    # baryon leaves (Lt=2 -> at most 2 chunks)
    w = dags.config_c3(N=12, Lt=2, S=64)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    _, roots, corr, st, ex = run_gpu(w, options={"h2d_chunk_bytes": 65536})
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)


def test_trace_fusion_on_off():
    """Traces fused into the GEMM that produces their later operand (partner tiles dotted
    with the output tile in registers) give the oracle's values, like the stand-alone trace
    items; ragged N (not a multiple of the 64-wide tile) exercises the zero-filled borders."""
    for (N, Lt) in ((40, 3), (64, 2), (96, 2)):
        w = dags.config_c2(N=N, Lt=Lt, n_loop4=70, n_loop2=6, n_corr=4)
        dag = Dag(w)
        r_or, c_or = values.run_workload(w, dag)
        res = {}
        for fuse in (1, 0):
            for dev in (False, True):
                _, roots, corr, st, ex = run_gpu(w, device_leaves=dev, options={"trace_fusion": fuse})
                assert_roots_close(roots, r_or)
                assert_corr_close(dag, r_or, corr, c_or)
                res[(fuse, dev)] = (roots, ex["n_kernels"])
        # fused: one more launch (the finish kernel summing tile partials)
        assert res[(1, True)][1] == res[(0, True)][1] + 1


def test_c3_nucleon_small():
    for (N, Lt, S) in ((8, 2, 4), (12, 2, 64), (20, 1, 64)):
        w = dags.config_c3(N=N, Lt=Lt, S=S)
        dag = Dag(w)
        r_or, c_or = values.run_workload(w, dag)
        for flags in (0, 16):
            _, roots, corr, st, ex = run_gpu(w, flags=flags)
            assert_roots_close(roots, r_or)
            assert_corr_close(dag, r_or, corr, c_or)


def test_c4_evictions_under_cap():
    """Two-baryon DAG with a capped pool: the plan evicts (leaves dropped, intermediates
    copied to pinned host and re-fetched); values still match the oracle."""
    w = dags.config_c4(N=8, Lt=1, S=4, n_trees=120, n_corr=4)
    dag = Dag(w)
    bary = 16 * 4 * 8 ** 3
    cap = 7 * bary
    order = tree.schedule(dag)
    p = lru.plan(dag, order, cap)
    assert p["evictions"] > 0 and p["d2h_count"] > 0
    r_or, c_or = values.run_workload(w, dag)
    for flags in (0, 1, 16):
        _, roots, corr, st, ex = run_gpu(w, cap=cap, flags=flags)
        assert st["evictions"] == p["evictions"] and st["h2d_bytes"] == p["h2d_bytes"]
        assert ex["d2h_bytes"] == p["d2h_bytes"] and ex["h2d_bytes"] == p["h2d_bytes"]
        assert_roots_close(roots, r_or)
        assert_corr_close(dag, r_or, corr, c_or)


def test_c4_next_use_evictions_under_cap():
    """The same capped two-baryon DAG with next-use eviction (reading E-9): the executed plan
    moves exactly the oracle's bytes (fewer than LRU) and the values still match."""
    w = dags.config_c4(N=8, Lt=1, S=4, n_trees=120, n_corr=4)
    dag = Dag(w)
    cap = 7 * 16 * 4 * 8 ** 3
    order = tree.schedule(dag)
    p = lru.plan(dag, order, cap, policy="next_use")
    assert p["evictions"] > 0
    assert p["h2d_bytes"] + p["d2h_bytes"] <= lru.plan(dag, order, cap)["h2d_bytes"] + lru.plan(dag, order, cap)["d2h_bytes"]
    r_or, c_or = values.run_workload(w, dag)
    for flags in (0, 16):
        _, roots, corr, st, ex = run_gpu(w, cap=cap, flags=flags, evict_next_use=True)
        assert st["evictions"] == p["evictions"] and ex["h2d_bytes"] == p["h2d_bytes"]
        assert ex["d2h_bytes"] == p["d2h_bytes"]
        assert_roots_close(roots, r_or)
        assert_corr_close(dag, r_or, corr, c_or)


def test_partitions_sum_to_whole():
    from paper_2511_02257_b200 import cc
    w = dags.config_c2(N=16, Lt=6, n_loop4=60, n_loop2=6, n_corr=4)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    for mode, n in ((cc.PART_TIME, 3), (cc.PART_TREES, 3)):
        total = {c: np.zeros(w.Lt, complex) for c in c_or}
        for p in range(n):
            _, roots, corr, st, ex = run_gpu(w, part=(n, p, mode))
            if mode == cc.PART_TIME:
                t0, t1 = partition.time_range(w.Lt, n, p)
                for c in corr:
                    total[c][t0:t1] += corr[c]
            else:
                for c in corr:
                    total[c] += corr[c]
        assert_corr_close(dag, r_or, total, c_or)


@pytest.mark.parametrize("flags", [0, 16])
def test_grid_parts_sum_to_whole(flags):
    """GRID split (reading M-2, 2 tree parts x 3 time parts): each part's correlator slices,
    placed at its time range and summed over tree parts, equal the whole DAG's."""
    w = dags.config_c2(N=16, Lt=6, n_loop4=60, n_loop2=6, n_corr=4)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    total = {c: np.zeros(w.Lt, complex) for c in c_or}
    for p in range(6):
        ctx, roots, corr, st, ex = run_gpu(w, part=("grid", 2, 3, p), flags=flags)
        t0, t1 = ctx.part_time_range()
        assert (t0, t1) == partition.time_range(w.Lt, 3, p % 3)
        for c in corr:
            total[c][t0:t1] += corr[c]
    assert_corr_close(dag, r_or, total, c_or)


def test_c2_full_size_sampled_slices():
    """BASELINE configs[1] at full size (N=128, Lt=64, 400 trees) in the bench's launch
    configuration (graph, device-resident leaves); the oracle computes time slices
    {0, 31, 63} only (per-slice independence is exact)."""
    w = dags.config_c2()
    dag = Dag(w)
    _, roots, corr, st, ex = run_gpu(w, flags=1, device_leaves=True, arena_mb=8192)
    for t in (0, 31, 63):
        r_or, c_or = values.run_workload(w, dag, t_range=(t, t + 1))
        assert_roots_close({k: v[t:t + 1] for k, v in roots.items()}, r_or)
        assert_corr_close(dag, r_or, {k: v[t:t + 1] for k, v in corr.items()}, c_or)


def test_stream_k_repeatable_bitwise(ctx):
    """Persistent stream-K: a tile split across CTAs is fixed up in a static order, so two
    launches give identical bits (also across problem sizes sharing the workspace)."""
    for (Lt, N, S, kind) in ((3, 100, 1, "mm1"), (1, 40, 64, "bb2"), (2, 8, 1, "mm1"), (1, 64, 16, "bb2")):
        if kind == "mm1":
            A = _random_phase((Lt, N, N), 11)
            B = _random_phase((Lt, N, N), 12)
            C1 = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
            C2 = torch.empty_like(C1)
            dA, dB = device_from(A), device_from(B)
            ctx.mm1(dA, dB, C1, Lt, N)
            ctx.mm1(dA, dB, C2, Lt, N)
            want = values.mm1(A, B)
            scale = np.matmul(np.abs(A), np.abs(B))
            shape = (Lt, N, N)
        else:
            A = _random_phase((Lt, S, N, N, N), 13)
            B = _random_phase((Lt, S, N, N, N), 14)
            C1 = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
            C2 = torch.empty_like(C1)
            dA, dB = device_from(A), device_from(B)
            ctx.bb2(dA, dB, C1, Lt, N, S)
            ctx.bb2(dA, dB, C2, Lt, N, S)
            want = values.bb2(A, B)
            scale = sum(np.matmul(np.abs(A[:, s]).reshape(Lt, N, N * N), np.abs(B[:, s]).reshape(Lt, N * N, N))
                        for s in range(S))
            shape = (Lt, N, N)
        torch.cuda.synchronize()
        g1, g2 = to_numpy_c(C1, shape), to_numpy_c(C2, shape)
        assert np.array_equal(g1, g2)
        assert np.all(np.abs(g1 - want) <= 1e-13 * scale)


def _oracle_tree_roots(w, dag, tree_ids, t):
    """Oracle roots of the given trees at time slice t only (their sub-DAGs, per-slice
    independence is exact)."""
    ops = {u: n.op for u, n in dag.nodes.items()}
    memo = {}

    def val(u):
        if u not in memo:
            n = dag.nodes[u]
            if not n.child:
                memo[u] = values.synthetic_leaf(w, u, ops[u], (t, t + 1))
            else:
                memo[u] = values.KERNELS[n.op](val(n.child[0]), val(n.child[1]))
        return memo[u]
    return {tr: val(dag.trees[tr][0]) for tr in tree_ids}


@pytest.mark.parametrize("N,n_pairs,n_trees", [(256, 120, 600), (512, 60, 200), (1024, 24, 60)])
def test_c5_large_N_time_part(N, n_pairs, n_trees):
    """c5 (MxM sweep, Lt=128) at N = 256 / 512 / 1024 as one rank's TIME part of an 8-GPU run
    (16 slices), leaves generated on the device by the bit-exact generator, bench launch
    configuration (graph replay); the oracle computes sampled trees at two of the part's slices."""
    from paper_2511_02257_b200 import cc
    w = dags.config_c5(N=N, Lt=128, n_pairs=n_pairs, n_trees=n_trees, n_corr=8)
    dag = Dag(w)
    arena = torch.empty(96 << 30, dtype=torch.uint8, device="cuda")
    ctx = cc.Context(0, arena)
    ctx.load_workload(w)
    ctx.partition(8, 5, cc.PART_TIME)
    t0, t1 = ctx.part_time_range()
    order, st = ctx.schedule(cc.CC_TREE)
    keep = []
    for u, n in dag.nodes.items():
        if n.child:
            continue
        per_t = N * N
        d = torch.empty(2 * (t1 - t0) * per_t, dtype=torch.float64, device="cuda")
        ctx.fill_synthetic(d, (t1 - t0) * per_t, w.data_seed, u, t0 * per_t, w.leaf_mode, srng.meson_sigma(N))
        keep.append(d)
        ctx.set_leaf_device(u, d)
    ctx.execute(1)
    ctx.execute(1)
    trees = ctx.part_trees()
    sample = trees[:: max(1, len(trees) // 6)][:6]
    for t in (t0, t1 - 1):
        want = _oracle_tree_roots(w, dag, sample, t)
        got = {tr: ctx.root_value(tr, t1 - t0)[t - t0:t - t0 + 1] for tr in sample}
        assert_roots_close(got, want)
    del arena
    torch.cuda.empty_cache()


def test_slice_major_baryon_chains_bitwise():
    """Slice-major item order with per-slice GEMM -> GEMM dependencies (BM1 -> BB2 -> TR, c3 /
    c4 shapes with Lt > 1, and the tritium chain BB1 -> BT2 -> BB1 -> BT2 -> BB3) gives values
    bit-identical to the op-major order and within tolerance of the oracle."""
    from paper_2511_02257_b200 import cc
    for w in (dags.config_c3(N=12, Lt=3, S=4), dags.config_c4(N=8, Lt=3, S=4, n_trees=20),
              dags.config_c6(N=8, Lt=3, S=4, n_trees=12)):
        dag = Dag(w)
        r_or = values.evaluate(dag, lambda u: values.synthetic_leaf(w, u, dag.nodes[u].op))
        for flags in (0, 1):
            a = run_gpu(w, flags=flags, device_leaves=bool(flags), options={"slice_major": 1})[1]
            b = run_gpu(w, flags=flags, device_leaves=bool(flags), options={"slice_major": 0})[1]
            for t in a:
                assert np.array_equal(a[t], b[t]), (w.name, flags, t)
            assert_roots_close(a, r_or)


def test_leaf_slots_placement_and_fallback():
    """Leaf slots (option leaf_slots): values bit-identical with and without, on the dataflow and
    op-by-op executors; a pool too small to hold every leaf next to the intermediates falls back
    to the shared placement (still exact)."""
    w = dags.config_c2(N=40, Lt=3, n_loop4=40, n_loop2=4, n_corr=3)
    dag = Dag(w)
    r_or = values.evaluate(dag, lambda u: values.synthetic_leaf(w, u, dag.nodes[u].op))
    for flags in (0, 16):
        a = run_gpu(w, flags=flags, options={"leaf_slots": 1})[1]
        b = run_gpu(w, flags=flags, options={"leaf_slots": 0})[1]
        for t in a:
            assert np.array_equal(a[t], b[t]), (flags, t)
        assert_roots_close(a, r_or)
    # an arena that holds the plan's peak but not every leaf slot next to it
    leaf_bytes = sum(dag.nodes[u].size for u, n in dag.nodes.items() if not n.child)
    from paper_2511_02257_b200 import cc
    scratch = cc.cc_scratch_bytes(w.Lt, w.N, w.S)
    peak = lru.plan(dag, tree.schedule(dag))["transient_peak"]
    arena_mb = max(1, int((scratch + peak + leaf_bytes // 2) * 1.05) >> 20) + 1
    ctx, roots, _, _, _ = run_gpu(w, arena_mb=arena_mb, options={"leaf_slots": 1})
    assert_roots_close(roots, r_or)


@pytest.mark.parametrize("flags", [0, 16])
def test_compaction_on_a_fragmented_pool(flags):
    """A two-baryon DAG under a cap in an arena whose pool best fit cannot place (fragmentation):
    cc_execute compacts with device-to-device moves (op by op), values match the oracle, the
    logical plan's copies are unchanged."""
    from paper_2511_02257_b200 import cc
    w = dags.config_c4(N=8, Lt=1, S=4, n_snk=4, n_src=4, n_mes=4, n_trees=40, seed=9)
    dag = Dag(w)
    baryon = 16 * 4 * 8 ** 3
    probe = cc.Context(-1)
    probe.load_workload(w)
    _, st = probe.schedule(cc.CC_TREE, cap_bytes=6 * baryon)
    pool = None
    for p in range((st["transient_peak"] + 1023) // 1024 * 1024, st["transient_peak"] * 5 // 4, 1024):
        fails = 0
        for nf in (False, True):                 # the executor tries next fit, then best fit
            try:
                probe.phys_plan(p, next_fit=nf)
            except cc.CCError:
                fails += 1
        if fails == 2:
            try:
                if probe.phys_plan(p, compact=True)["n_moves"] > 0:
                    pool = p
                    break
            except cc.CCError:
                pass
    assert pool is not None
    # an arena of exactly scratch + pool bytes (the scratch depends on the arena size through the
    # Ozaki workspace: iterate to the fixed point)
    size = 64 << 20
    for _ in range(8):
        arena = torch.empty(size, dtype=torch.uint8, device="cuda")
        ctx = cc.Context(0, arena)
        ctx.load_workload(w)
        ctx.schedule(cc.CC_TREE, cap_bytes=6 * baryon)
        want = ctx.scratch_of() + pool
        if want == size:
            break
        size = want
    assert want == size
    _, roots, corr, st2, ex = run_gpu(w, cap=6 * baryon, flags=flags, ctx=ctx)
    r_or = values.evaluate(dag, lambda u: values.synthetic_leaf(w, u, dag.nodes[u].op))
    assert_roots_close(roots, r_or)
    assert ex["move_bytes"] > 0
    # the dataflow flags start up to 4 leading leaf copies before the physical plan exists; a
    # compacting plan runs op by op and copies them again (counted: they crossed PCIe)
    assert ex["d2h_bytes"] == st2["d2h_bytes"]
    assert st2["h2d_bytes"] <= ex["h2d_bytes"] <= st2["h2d_bytes"] + (4 * 16 * 4 * 8 ** 3 if flags == 0 else 0)


def test_trace_runs_with_refetched_leaves_under_cap():
    """Leaf-reading traces under a cap that evicts and re-fetches leaves: H2D copies sit between
    traces in the dataflow order (a copy waits for the traces reading the memory it overwrites,
    the next traces wait for the copy), so trace runs must break at copies (3a').  Values vs the
    oracle on the dataflow worker, trace runs on and off, stream and graph."""
    w = dags.config_c2(N=16, Lt=2, n_loop4=10, n_loop2=60, n_corr=3)
    dag = Dag(w)
    cap = 6 * 2 * 16 * 16 * 16
    p = lru.plan(dag, tree.schedule(dag), cap)
    assert p["evictions"] > 0 and p["h2d_count"] > 32
    r_or, c_or = values.run_workload(w, dag)
    for tg in (1, 0):
        for flags in (0, 1):
            _, roots, corr, st, ex = run_gpu(w, cap=cap, flags=flags, options={"trace_groups": tg})
            assert st["evictions"] == p["evictions"] and ex["h2d_bytes"] == p["h2d_bytes"]
            assert_roots_close(roots, r_or)
            assert_corr_close(dag, r_or, corr, c_or)


def test_trace_runs_bit_identical():
    """Trace runs (option trace_groups) only reorder work items: roots are bit-identical with the
    option off, on a slice-major plan (c2-shaped) and on an op-major plan with split traces
    (c5-shaped at N = 256: 4 pieces per slice through the partial ring, memory reuse)."""
    for w, arena in ((dags.config_c2(N=40, Lt=4, n_loop4=60, n_loop2=6, n_corr=3), 256),
                     (dags.config_c5(N=256, Lt=3, n_mes=8, n_pairs=20, n_trees=120, n_corr=3), 1024)):
        dag = Dag(w)
        r_or, _ = values.run_workload(w, dag)
        got = []
        for tg in (0, 1):
            _, roots, corr, st, ex = run_gpu(w, flags=0, arena_mb=arena, options={"trace_groups": tg})
            assert_roots_close(roots, r_or)
            got.append(roots)
        for t in r_or:
            assert np.array_equal(got[0][t], got[1][t]), t


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_dataflow_random_dags_under_caps(seed):
    """Randomised c2-shaped DAGs (ragged N, few slices) through the dataflow worker, unbounded and
    under a cap that evicts and re-fetches leaves: trace runs, copy order and slice-major items
    must keep the queues topological (no hang) and the values exact (oracle)."""
    r = np.random.default_rng(seed)
    N = int(r.choice([24, 40, 56]))
    Lt = int(r.integers(2, 4))
    w = dags.config_c2(N=N, Lt=Lt, n_loop4=int(r.integers(20, 60)), n_loop2=int(r.integers(4, 30)), n_corr=3,
                       seed=seed)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    leaf = Lt * N * N * 16
    for cap in (0, 8 * leaf):
        p = lru.plan(dag, tree.schedule(dag), cap) if cap else None
        _, roots, corr, st, ex = run_gpu(w, cap=cap, flags=0)
        if p is not None:
            assert st["evictions"] == p["evictions"] and ex["h2d_bytes"] == p["h2d_bytes"]
        assert_roots_close(roots, r_or)
        assert_corr_close(dag, r_or, corr, c_or)
