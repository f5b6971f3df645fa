"""GPU parity of the engines cc_execute actually runs, on the data the tolerance argument is
hardest on (reading V-4): random-phase leaves through every executor, closed-form exact
correlators with complex coefficients, and the full-size c3 / c4 shapes (BB2 at K = S N^2 = 2^20,
SURVEY V-4's worst case) against the oracle on sampled time slices / trees.

Tolerances (V-4): phase-limited data, per root |gpu - oracle| <= 1e-10 |oracle|; random-phase
data, per root |gpu - oracle| <= 1e-10 R_abs, where R_abs is the same DAG evaluated by the
oracle on |leaf| values (every product and sum of the contraction chain taken in absolute
value: the standard bound of any summation order's rounding error is a multiple of u R_abs);
correlators against sum_terms |coef| R_abs (or |coef root| for phase-limited data).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import dags, rng as srng  # noqa: E402
from oracle import values, lru, tree  # noqa: E402
from oracle.dag import Dag  # noqa: E402
from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close, device_from, to_numpy_c  # noqa: E402
from test_oracle_values import scaled_ones_scalars, scaled_ones_factor  # noqa: E402

ENGINES = [0, 1, 16, 17, 64, 128]   # dataflow stream / graph, op-by-op stream / graph, Ozaki, AUTO


def _abs_roots(dag, leaf):
    """R_abs: the DAG evaluated on |leaf| (all arithmetic on non-negative values)."""
    return values.evaluate(dag, lambda u: np.abs(leaf(u)).astype(np.complex128))


def _check_scaled(got_roots, got_corr, dag, r_or, c_or, r_abs, rel=1e-10):
    for t, want in r_or.items():
        err = np.abs(got_roots[t] - want)
        assert np.all(err <= rel * np.abs(r_abs[t])), (t, float(np.max(err / np.abs(r_abs[t]))))
    scale = {}
    for (c, t, coef) in dag.terms:
        scale[c] = scale.get(c, 0.0) + np.abs(coef) * np.abs(r_abs[t])
    for c, want in c_or.items():
        assert np.all(np.abs(got_corr[c] - want) <= rel * scale[c]), c


@pytest.mark.parametrize("flags", ENGINES)
def test_random_phase_dag_every_engine(flags):
    """A c2-shaped DAG (ragged N = 72: two 64-wide tiles, the second partial) with random-phase
    leaves (both signs, cancellation in every sum) and Gaussian-integer coefficients through
    every executor, including the default dataflow worker's 3M k-tiles (reading V-3)."""
    w = dags.config_c2(N=72, Lt=3, n_loop4=60, n_loop2=6, n_corr=4, coefs="complex")
    w.leaf_mode = srng.MODE_RANDOM_PHASE
    dag = Dag(w)
    ops = {u: n.op for u, n in dag.nodes.items()}
    leaf = lambda u: values.synthetic_leaf(w, u, ops[u])   # noqa: E731
    r_or = values.evaluate(dag, leaf)
    c_or = values.correlators(dag, r_or)
    r_abs = _abs_roots(dag, leaf)
    _, roots, corr, st, ex = run_gpu(w, flags=flags, arena_mb=512)
    _check_scaled(roots, corr, dag, r_or, c_or, r_abs)


@pytest.mark.parametrize("flags", ENGINES)
def test_random_phase_baryon_dag_every_engine(flags):
    """c4-shaped two-baryon DAG (BM1 dressings, BB2 over spin, traces) with random-phase leaves
    and a capped pool (evictions, D2H and re-fetches) through every executor."""
    w = dags.config_c4(N=12, Lt=2, S=8, n_snk=3, n_src=3, n_mes=4, n_trees=40, n_corr=3)
    w.leaf_mode = srng.MODE_RANDOM_PHASE
    dag = Dag(w)
    ops = {u: n.op for u, n in dag.nodes.items()}
    leaf = lambda u: values.synthetic_leaf(w, u, ops[u])   # noqa: E731
    r_or = values.evaluate(dag, leaf)
    c_or = values.correlators(dag, r_or)
    r_abs = _abs_roots(dag, leaf)
    cap = 6 * 16 * 2 * 8 * 12 ** 3
    p = lru.plan(dag, tree.schedule(dag), cap)
    assert p["evictions"] > 0
    _, roots, corr, st, ex = run_gpu(w, flags=flags, cap=cap, arena_mb=256)
    assert st["evictions"] == p["evictions"]
    assert ex["h2d_bytes"] == p["h2d_bytes"] and ex["d2h_bytes"] == p["d2h_bytes"]
    _check_scaled(roots, corr, dag, r_or, c_or, r_abs)


@pytest.mark.parametrize("flags", ENGINES)
def test_closed_form_exact_correlators(flags):
    """Leaves c_u J: every root and every correlator (Gaussian-integer coefficients) is an exact
    integer (test_oracle_values.scaled_ones_scalars); every engine reproduces them bit for bit."""
    N, Lt = 40, 2
    w = dags.config_c2(N=N, Lt=Lt, n_loop4=50, n_loop2=5, n_corr=4, coefs="complex")
    sc = scaled_ones_scalars(w)
    _, roots, corr, st, ex = run_gpu(
        w, flags=flags, leaf_fn=lambda u, op: scaled_ones_factor(u) * np.ones((Lt, N, N), complex))
    root_of = dict(w.trees)
    want = {}
    for (c, t, re, im) in w.terms:
        r = sc[root_of[t]]
        a, b = want.get(c, (0, 0))
        want[c] = (a + int(re) * r, b + int(im) * r)
    for t, r in root_of.items():
        assert np.array_equal(roots[t], np.full(Lt, complex(sc[r], 0))), t
    for c, (a, b) in want.items():
        assert np.array_equal(corr[c], np.full(Lt, complex(a, b))), c


def test_runtime_copy_counts_match_plan():
    """cc_exec_stats h2d/d2h bytes are counted as the executor enqueues copies: equal to the
    oracle plan's bytes on every executor (a dropped or duplicated copy would show)."""
    w = dags.config_c4(N=8, Lt=1, S=4, n_trees=120, n_corr=4)
    dag = Dag(w)
    cap = 7 * 16 * 4 * 8 ** 3
    for nu in (False, True):
        p = lru.plan(dag, tree.schedule(dag), cap, policy="next_use" if nu else "lru")
        for flags in (0, 16, 17, 64):
            ctx, roots, corr, st, ex = run_gpu(w, cap=cap, flags=flags, evict_next_use=nu)
            assert (ex["h2d_bytes"], ex["d2h_bytes"]) == (p["h2d_bytes"], p["d2h_bytes"]), (nu, flags)
    # device-resident leaves: nothing copied
    _, _, _, st, ex = run_gpu(dags.config_c1(), device_leaves=True)
    assert ex["h2d_bytes"] == 0 and ex["d2h_bytes"] == 0


def _pinned_leaf(w, u, op, mode=None):
    shape = values.leaf_shape(op, w.Lt, w.N, w.S)
    sigma = srng.meson_sigma(w.N) if op == dags.LEAF_M else srng.baryon_sigma(w.N, w.S)
    h = torch.empty(int(np.prod(shape)) * 2, dtype=torch.float64, pin_memory=True)
    srng.leaf_values_into(h.numpy().view(np.complex128), w.data_seed, u, 0, sigma,
                          w.leaf_mode if mode is None else mode)
    return h


def _oracle_trees(w, dag, tree_ids, host, t_range=None):
    """Oracle roots of some trees from the leaves' host copies (one slice range)."""
    memo = {}

    def val(u):
        if u not in memo:
            n = dag.nodes[u]
            if not n.child:
                shape = values.leaf_shape(n.op, w.Lt, w.N, w.S)
                full = host[u].numpy().view(np.complex128).reshape(shape)
                memo[u] = full if t_range is None else full[t_range[0]:t_range[1]]
            else:
                memo[u] = values.KERNELS[n.op](val(n.child[0]), val(n.child[1]))
        return memo[u]
    return {t: val(dag.trees[t][0]) for t in tree_ids}


@pytest.mark.parametrize("flags", [0, 64])
def test_c4_full_shape_bb2_K_2e20(flags):
    """c4 at its full shapes (N = 128, S = 64, Lt = 1: 2 GiB baryon leaves, BB2 with K = 2^20) on
    a handful of trees, leaves in pinned host memory, pool capped at 4 baryons (3 evictions, a D2H
    of a 2 GiB dressing, re-fetches), on the DMMA dataflow worker and the Ozaki engine; the oracle
    evaluates two sampled trees (values within 1e-10 relative, phase-limited data) and the plan's
    integers.  DESIGN V-4 / V-6: the K = 2^20 error bound at 5 Ozaki slices."""
    w = dags.config_c4(N=128, Lt=1, S=64, n_snk=2, n_src=2, n_mes=4, n_trees=6, n_corr=2, seed=3)
    dag = Dag(w)
    host = {u: _pinned_leaf(w, u, n.op) for u, n in dag.nodes.items() if not n.child}
    bary = 16 * 64 * 128 ** 3
    cap = 4 * bary
    p = lru.plan(dag, tree.schedule(dag), cap)
    assert p["evictions"] > 0 and p["d2h_count"] > 0
    _, roots, corr, st, ex = run_gpu(w, flags=flags, cap=cap, arena_mb=int(6.5 * bary) >> 20,
                                     leaf_fn=lambda u, op: host[u])
    assert (st["evictions"], st["h2d_bytes"], st["d2h_bytes"]) == (p["evictions"], p["h2d_bytes"], p["d2h_bytes"])
    assert (ex["h2d_bytes"], ex["d2h_bytes"]) == (p["h2d_bytes"], p["d2h_bytes"])
    # two sampled trees: the first and the one with the most dressings (BM1 -> BB2 chains)
    def n_bm1(t):
        return sum(1 for u in dag.trees[t][1] if dag.nodes[u].op == dags.BM1)
    sample = sorted({dag.tree_ids[0], max(dag.tree_ids, key=n_bm1)})
    want = _oracle_trees(w, dag, sample, host)
    assert_roots_close({t: roots[t] for t in sample}, want)


@pytest.mark.parametrize("engine", ["dmma", "ozaki"])
def test_bb2_K_2e20_random_phase(engine):
    """One c4-shaped BB2 (N = 128, S = 64: K = 2^20, 2 GiB operands) on random-phase data, both
    engines, against the oracle within 1e-10 of the |A||B| scale (the worst case of V-4)."""
    from paper_2511_02257_b200 import cc
    N, S, Lt = 128, 64, 1
    shape = (Lt, S, N, N, N)
    A = np.empty(shape, complex)
    B = np.empty(shape, complex)
    sig = srng.baryon_sigma(N, S)
    srng.leaf_values_into(A, 7, 101, 0, sig, srng.MODE_RANDOM_PHASE)
    srng.leaf_values_into(B, 7, 102, 0, sig, srng.MODE_RANDOM_PHASE)
    ctx = cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
    dA, dB = device_from(A), device_from(B)
    C = torch.empty(Lt * N * N * 2, dtype=torch.float64, device="cuda")
    if engine == "dmma":
        ctx.bb2(dA, dB, C, Lt, N, S)
    else:
        ws = torch.empty(cc.cc_gemm_ozaki_workspace_bytes(cc.CC_BB2, Lt, N, S, 5), dtype=torch.uint8, device="cuda")
        ctx.gemm_ozaki(cc.CC_BB2, dA, dB, C, Lt, N, S, 5, ws)
    torch.cuda.synchronize()
    got = to_numpy_c(C, (Lt, N, N))
    del dA, dB
    want = values.bb2(A, B)
    scale = values.bb2(np.abs(A).astype(complex), np.abs(B).astype(complex)).real
    err = np.abs(got - want) / scale
    assert float(err.max()) <= 1e-10, float(err.max())


@pytest.mark.parametrize("flags", [0, 64])
def test_c3_full_size_sampled_slices(flags):
    """c3 at full size (N = 64, S = 64, Lt = 32: two 8 GiB baryon leaves, BM1 then BB2 with
    K = 2^18, then the trace), leaves device-resident (generated by the oracle's generator, copied
    in), on the dataflow worker and the Ozaki engine; the oracle evaluates slices 0 and 31."""
    w = dags.config_c3()
    dag = Dag(w)
    host = {u: _pinned_leaf(w, u, n.op) for u, n in dag.nodes.items() if not n.child}
    dev = {u: h.to("cuda") for u, h in host.items()}
    from paper_2511_02257_b200 import cc
    ctx = cc.Context(0, torch.empty(20 << 30, dtype=torch.uint8, device="cuda"))
    ctx.load_workload(w)
    ctx.schedule(cc.CC_TREE)
    for u, d in dev.items():
        ctx.set_leaf_device(u, d)
    ctx.execute(flags)
    got = ctx.root_value(0, w.Lt)
    for t in (0, 31):
        r = _oracle_trees(w, dag, [0], host, t_range=(t, t + 1))
        assert_roots_close({0: got[t:t + 1]}, r)


@pytest.mark.parametrize("N", [36, 56, 136])
def test_trace_stage_box_paths(N):
    """The worker's TR_MM stages load each 32x32 operand block as one chunk-wide TMA box when
    N % 8 == 0 (56: ragged blocks with zero-filled chunks and rows; 136: past one 128-row
    block) and as four 32-row boxes otherwise (36); random-phase leaves against R_abs."""
    w = dags.config_c2(N=N, Lt=2, n_loop4=24, n_loop2=4, n_corr=3, coefs="complex")
    w.leaf_mode = srng.MODE_RANDOM_PHASE
    dag = Dag(w)
    ops = {u: n.op for u, n in dag.nodes.items()}
    leaf = lambda u: values.synthetic_leaf(w, u, ops[u])   # noqa: E731
    r_or = values.evaluate(dag, leaf)
    c_or = values.correlators(dag, r_or)
    r_abs = _abs_roots(dag, leaf)
    for flags in (0, 1):
        _, roots, corr, st, ex = run_gpu(w, flags=flags, arena_mb=512)
        _check_scaled(roots, corr, dag, r_or, c_or, r_abs)
