"""GPU parity of the tritium-class BxBxB kinds (readings T4-1..T4-4):
BB1 (baryon x baryon single index -> tetraquark N^4 node), BT2 (baryon x tetra double index ->
baryon), BB3 (baryon x baryon contract-all), stand-alone and inside whole c6 DAGs through every
executor, against the oracle (tolerances as tests/test_gpu_parity_engines.py, reading V-4)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import dags, rng as srng  # noqa: E402
from oracle import values, lru, tree  # noqa: E402
from oracle.dag import Dag  # noqa: E402
from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close, device_from, to_numpy_c  # noqa: E402
from test_gpu_parity_engines import ENGINES, _abs_roots, _check_scaled  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_02257_b200 import cc
    return cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))


def _vals(shape, seed, mode=srng.MODE_PHASE_LIMITED, sigma=1.0):
    n = int(np.prod(shape))
    return srng.leaf_values(seed, 3000 + seed, 0, n, sigma, mode).reshape(shape)


def _run(ctx, kind, A, B, Lt, N, S, engine="dmma"):
    from paper_2511_02257_b200 import cc
    shape = {"bb1": (Lt, N, N, N, N), "bt2": (Lt, S, N, N, N), "bb3": (Lt,)}[kind]
    out = torch.full((int(np.prod(shape)) * 2,), float("nan"), dtype=torch.float64, device="cuda")
    dA, dB = device_from(A), device_from(B)
    if engine == "dmma":
        getattr(ctx, kind)(dA, dB, out, Lt, N, S)
    else:
        op = {"bb1": cc.CC_BB1, "bt2": cc.CC_BT2}[kind]
        ws = torch.empty(cc.cc_gemm_ozaki_workspace_bytes(op, Lt, N, S, 5), dtype=torch.uint8, device="cuda")
        ctx.gemm_ozaki(op, dA, dB, out, Lt, N, S, 5, ws)
    torch.cuda.synchronize()
    return to_numpy_c(out, shape)


@pytest.mark.parametrize("engine", ["dmma", "ozaki"])
@pytest.mark.parametrize("Lt,N,S", [(2, 4, 2), (1, 8, 4), (2, 12, 8), (1, 20, 3), (1, 32, 64), (2, 33, 2)])
def test_bb1_bt2_elementwise(ctx, engine, Lt, N, S):
    sb = srng.baryon_sigma(N, S)
    A = _vals((Lt, S, N, N, N), 1, sigma=sb)
    B = _vals((Lt, S, N, N, N), 2, sigma=sb)
    X = _vals((Lt, N, N, N, N), 3, sigma=1.0 / N ** 2)
    for kind, L, R, ref in (("bb1", A, B, values.bb1), ("bt2", A, X, values.bt2)):
        got = _run(ctx, kind, L, R, Lt, N, S, engine)
        want = ref(L, R)
        err = float(np.max(np.abs(got - want) / np.abs(want)))
        assert err <= 1e-10, (kind, err)


@pytest.mark.parametrize("Lt,N,S", [(2, 4, 2), (3, 8, 4), (1, 32, 64), (2, 33, 3), (1, 64, 8)])
def test_bb3_elementwise(ctx, Lt, N, S):
    sb = srng.baryon_sigma(N, S)
    A = _vals((Lt, S, N, N, N), 4, sigma=sb)
    B = _vals((Lt, S, N, N, N), 5, sigma=sb)
    got = _run(ctx, "bb3", A, B, Lt, N, S)
    want = values.bb3(A, B)
    assert float(np.max(np.abs(got - want) / np.abs(want))) <= 1e-10


@pytest.mark.parametrize("engine", ["dmma", "ozaki"])
def test_bxbxb_random_phase_and_closed_forms(ctx, engine):
    """Random-phase data against the |A||B| scale; all-ones closed forms exactly (BB1 = S N J_T,
    BT2 = N^2 J_B, BB3 = S N^3)."""
    Lt, N, S = 2, 16, 8
    A = _vals((Lt, S, N, N, N), 6, srng.MODE_RANDOM_PHASE)
    B = _vals((Lt, S, N, N, N), 7, srng.MODE_RANDOM_PHASE)
    X = _vals((Lt, N, N, N, N), 8, srng.MODE_RANDOM_PHASE)
    for kind, L, R, ref in (("bb1", A, B, values.bb1), ("bt2", A, X, values.bt2)):
        got = _run(ctx, kind, L, R, Lt, N, S, engine)
        scale = ref(np.abs(L).astype(complex), np.abs(R).astype(complex)).real
        assert np.all(np.abs(got - ref(L, R)) <= 1e-10 * scale), kind
    JB = np.ones((Lt, S, N, N, N), complex)
    JT = np.ones((Lt, N, N, N, N), complex)
    assert np.array_equal(_run(ctx, "bb1", JB, JB, Lt, N, S, engine), S * N * JT)
    assert np.array_equal(_run(ctx, "bt2", JB, JT, Lt, N, S, engine), N * N * JB)
    if engine == "dmma":
        got = _run(ctx, "bb3", A, B, Lt, N, S)
        scale = values.bb3(np.abs(A).astype(complex), np.abs(B).astype(complex)).real
        assert np.all(np.abs(got - values.bb3(A, B)) <= 1e-10 * scale)
        assert np.array_equal(_run(ctx, "bb3", JB, JB, Lt, N, S), np.full(Lt, S * N ** 3, complex))


@pytest.mark.parametrize("flags", ENGINES)
def test_c6_dag_every_engine(flags):
    """A tritium-like c6 DAG (families with BB1 -> BT2 -> BB1 -> BT2 -> BB3 chains and
    BB2 / TR_MM meson branches; tetra, baryon and meson nodes) through every executor, phase-
    limited leaves, per root relative 1e-10 and correlators against sum |coef root|."""
    w = dags.config_c6(N=10, Lt=2, S=4, n_trees=60, n_corr=3, coefs="complex")
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    _, roots, corr, st, ex = run_gpu(w, flags=flags, arena_mb=256)
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)


@pytest.mark.parametrize("flags", [0, 16, 64])
def test_c6_random_phase_capped(flags):
    """The same with random-phase leaves and a pool capped below the plan's peak (evictions of
    tetra and baryon intermediates: D2H + re-fetch); the executed bytes equal the oracle plan."""
    w = dags.config_c6(N=8, Lt=2, S=4, n_trees=40, n_corr=2)
    w.leaf_mode = srng.MODE_RANDOM_PHASE
    dag = Dag(w)
    ops = {u: n.op for u, n in dag.nodes.items()}
    leaf = lambda u: values.synthetic_leaf(w, u, ops[u])   # noqa: E731
    r_or = values.evaluate(dag, leaf)
    c_or = values.correlators(dag, r_or)
    r_abs = _abs_roots(dag, leaf)
    bary = 16 * 2 * 4 * 8 ** 3
    cap = 6 * bary
    p = lru.plan(dag, tree.schedule(dag), cap)
    assert p["evictions"] > 0 and p["d2h_count"] > 0
    _, roots, corr, st, ex = run_gpu(w, flags=flags, cap=cap, arena_mb=256)
    assert (ex["h2d_bytes"], ex["d2h_bytes"]) == (p["h2d_bytes"], p["d2h_bytes"])
    _check_scaled(roots, corr, dag, r_or, c_or, r_abs)


@pytest.mark.parametrize("flags", [0, 64])
def test_c6_tritium_size_sampled(flags):
    """c6 at the paper's tritium size class (N = 32, S = 64: 32 MiB baryon and 16 MiB tetra
    slices), Lt = 4, leaves device-resident (generated by the shared generator on the host),
    oracle on sampled trees at slices 0 and 3."""
    from paper_2511_02257_b200 import cc
    w = dags.config_c6(N=32, Lt=4, S=64, n_trees=24, n_corr=3)
    dag = Dag(w)
    host = {}
    for u, n in dag.nodes.items():
        if not n.child:
            host[u] = np.empty(values.leaf_shape(n.op, w.Lt, w.N, w.S), complex)
            srng.leaf_values_into(host[u], w.data_seed, u, 0, srng.baryon_sigma(w.N, w.S))
    dev = {u: device_from(h) for u, h in host.items()}
    ctx = cc.Context(0, torch.empty(8 << 30, dtype=torch.uint8, device="cuda"))
    ctx.load_workload(w)
    ctx.schedule(cc.CC_TREE)
    for u, d in dev.items():
        ctx.set_leaf_device(u, d)
    ctx.execute(flags)
    sample = dag.tree_ids[:: max(1, len(dag.tree_ids) // 4)][:4]
    for t in (0, 3):
        memo = {}

        def val(u):
            if u not in memo:
                nd = dag.nodes[u]
                memo[u] = host[u][t:t + 1] if not nd.child else values.KERNELS[nd.op](val(nd.child[0]), val(nd.child[1]))
            return memo[u]
        want = {tr: val(dag.trees[tr][0]) for tr in sample}
        got = {tr: ctx.root_value(tr, w.Lt)[t:t + 1] for tr in sample}
        assert_roots_close(got, want)
