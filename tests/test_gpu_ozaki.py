"""GPU parity of the tcgen05 INT8 path (DESIGN reading V-6).

- cc_i8gemm_tn: the UMMA descriptor / TMEM machinery alone, bit-exact against an integer
  matmul (numpy int64).
- cc_mm1_ozaki: MM1 by Ozaki splitting, against the oracle's MM1 (oracle/values.py, numpy
  complex128): phase-limited data within 1e-10 relative per element (north_star), random-phase
  data within 1e-10 of the |A||B| error scale (V-4), all-ones closed form exactly (N J).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import rng as srng  # noqa: E402
from oracle import values  # noqa: E402
from gpu_helpers import device_from, to_numpy_c  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_02257_b200 import cc
    return cc.Context(0, torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))


@pytest.mark.parametrize("M,Nn,K", [(128, 192, 64), (256, 192, 192), (128, 384, 512), (384, 192, 1024)])
def test_i8gemm_bit_exact(ctx, M, Nn, K):
    g = np.random.default_rng(M * 7 + Nn + K)
    A = g.integers(-127, 128, size=(M, K), dtype=np.int8)
    B = g.integers(-127, 128, size=(Nn, K), dtype=np.int8)
    A[0, :] = 127                      # extreme rows/cols: |sum| = 127^2 K
    B[0, :] = -127
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.zeros((M, Nn), dtype=torch.int32, device="cuda")
    ctx.i8gemm_tn(dA, dB, dC, M, Nn, K)
    want = A.astype(np.int64) @ B.astype(np.int64).T
    got = dC.cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)


def _phase_limited(shape, seed):
    n = int(np.prod(shape))
    return srng.leaf_values(seed, 3000 + seed, 0, n, 1.0).reshape(shape)


def _random_phase(shape, seed):
    n = int(np.prod(shape))
    return srng.leaf_values(seed, 4000 + seed, 0, n, 1.0, srng.MODE_RANDOM_PHASE).reshape(shape)


def _run(ctx, A, B, Lt, N, s):
    from paper_2511_02257_b200 import cc
    ws = torch.empty(cc.cc_mm1_ozaki_workspace_bytes(Lt, N, s), dtype=torch.uint8, device="cuda")
    C = torch.full((Lt * N * N * 2,), float("nan"), dtype=torch.float64, device="cuda")
    ctx.mm1_ozaki(device_from(A), device_from(B), C, Lt, N, s, ws)
    torch.cuda.synchronize()
    return to_numpy_c(C, (Lt, N, N))


@pytest.mark.parametrize("Lt,N", [(1, 8), (2, 33), (3, 64), (2, 100), (4, 128), (1, 200), (2, 256), (1, 512)])
@pytest.mark.parametrize("s", [5, 6])
def test_mm1_ozaki_phase_limited(ctx, Lt, N, s):
    A = _phase_limited((Lt, N, N), 1 + N)
    B = _phase_limited((Lt, N, N), 2 + N)
    got = _run(ctx, A, B, Lt, N, s)
    want = values.mm1(A, B)
    err = float(np.max(np.abs(got - want) / np.abs(want)))
    assert err <= 1e-10, err


@pytest.mark.parametrize("Lt,N", [(2, 48), (1, 130), (1, 256)])
def test_mm1_ozaki_random_phase_scale(ctx, Lt, N):
    A = _random_phase((Lt, N, N), 5)
    B = _random_phase((Lt, N, N), 6)
    A[0, 3, :] *= 1e-3                   # a row and a column far below the others' scale
    B[0, :, 5] *= 1e6
    got = _run(ctx, A, B, Lt, N, 5)
    want = values.mm1(A, B)
    scale = np.matmul(np.abs(A), np.abs(B))
    assert np.all(np.abs(got - want) <= 1e-10 * scale)


def test_mm1_ozaki_closed_form_all_ones(ctx):
    Lt, N = 2, 96
    J = np.ones((Lt, N, N), dtype=np.complex128)
    for s in (4, 5, 7):
        got = _run(ctx, J, J, Lt, N, s)
        assert np.array_equal(got, N * J)
    Z = np.zeros_like(J)                 # a zero operand (exponent 0, all-zero slices)
    assert np.array_equal(_run(ctx, Z, J, Lt, N, 5), Z)
    M = -J                               # -1 -> top digit -32 (after scaling by 2^-1), zeros below
    assert np.array_equal(_run(ctx, M, J, Lt, N, 5), -N * J)


@pytest.mark.parametrize("flags", [64, 65])
def test_executor_ozaki_mm1_c2_small(flags):
    """cc_execute with every MM1 on the Ozaki engine (flags bit 6; +bit 0 = CUDA graph):
    roots within 1e-10 of the oracle, correlators within 1e-10 of sum|coef root|."""
    from synth import dags
    from oracle.dag import Dag
    from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close
    w = dags.config_c2(N=72, Lt=3, n_loop4=60, n_loop2=6, n_corr=4)
    dag = Dag(w)
    _, roots, corr, st, ex = run_gpu(w, flags=flags)
    r_or, c_or = values.run_workload(w, dag)
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)


def test_executor_ozaki_mm1_c5_time_part_deterministic():
    """c5-shaped DAG (N=256) on one TIME part with the Ozaki MM1 engine: oracle parity and
    bit-identical roots over two executes (fixed-order reductions, no atomics on values)."""
    from synth import dags
    from oracle.dag import Dag
    from oracle.partition import time_range
    from paper_2511_02257_b200 import cc
    from gpu_helpers import run_gpu, assert_roots_close
    w = dags.config_c5(N=256, Lt=8, n_pairs=40, n_trees=120, n_corr=4)
    dag = Dag(w)
    ctx, roots, corr, st, ex = run_gpu(w, flags=64, part=(4, 1, cc.PART_TIME), arena_mb=2048, device_leaves=True)
    t0, t1 = time_range(w.Lt, 4, 1)
    r_or, _ = values.run_workload(w, dag, t_range=(t0, t1))
    assert_roots_close({k: roots[k] for k in r_or}, r_or)
    ctx.execute(64)
    again = {t: ctx.root_value(t, t1 - t0) for t in roots}
    assert all(np.array_equal(again[t], roots[t]) for t in roots)


def test_mm1_ozaki_error_margin_large_N(ctx):
    """N=1024 with the executor's 5 slices: the balanced digits keep the error ~1e-13, two orders
    of magnitude inside the 1e-10 bar (V-6); 4 slices (30 bits) must be visibly worse — the
    slice count, not an accident of the data, is what meets the bar."""
    Lt, N = 1, 1024
    A = _phase_limited((Lt, N, N), 77)
    B = _phase_limited((Lt, N, N), 78)
    want = values.mm1(A, B)
    err5 = float(np.max(np.abs(_run(ctx, A, B, Lt, N, 5) - want) / np.abs(want)))
    err4 = float(np.max(np.abs(_run(ctx, A, B, Lt, N, 4) - want) / np.abs(want)))
    assert err5 <= 1e-11, err5
    assert err4 > 10 * err5, (err4, err5)


def test_executor_ozaki_leaf_form_cache_bitwise():
    """Leaves split once per execute and shared by their MM1s (cache in the free pool above the
    plan's high water) give bit-identical roots to splitting per MM1 (option ozaki_leaf_cache=0):
    the slices are a deterministic function of the leaf."""
    from synth import dags
    from oracle.dag import Dag
    from gpu_helpers import run_gpu, assert_roots_close
    w = dags.config_c2(N=64, Lt=4, n_loop4=50, n_loop2=4, n_corr=3)
    dag = Dag(w)
    ctx, roots, corr, st, ex = run_gpu(w, flags=64, arena_mb=512)
    r_or, _ = values.run_workload(w, dag)
    assert_roots_close(roots, r_or)
    ctx.set_options(ozaki_leaf_cache=0)
    ctx.execute(64)
    again = {t: ctx.root_value(t, w.Lt) for t in roots}
    assert all(np.array_equal(again[t], roots[t]) for t in roots)


def _run_gemm(ctx, op, A, B, Lt, N, S, s, out_shape, ws_bytes=None):
    from paper_2511_02257_b200 import cc
    full = cc.cc_gemm_ozaki_workspace_bytes(op, Lt, N, S, s)
    ws = torch.empty(ws_bytes or full, dtype=torch.uint8, device="cuda")
    C = torch.full((int(np.prod(out_shape)) * 2,), float("nan"), dtype=torch.float64, device="cuda")
    ctx.gemm_ozaki(op, device_from(A), device_from(B), C, Lt, N, S, s, ws)
    torch.cuda.synchronize()
    return to_numpy_c(C, out_shape)


@pytest.mark.parametrize("Lt,N,S", [(2, 8, 4), (1, 12, 64), (2, 16, 8), (1, 33, 2), (3, 24, 16)])
def test_bm1_ozaki(ctx, Lt, N, S):
    """BM1 (baryon x meson, M = S N^2 rows) on the Ozaki engine vs the oracle's BM1."""
    from paper_2511_02257_b200 import cc
    A = _phase_limited((Lt, S, N, N, N), 10 + N)
    M = _phase_limited((Lt, N, N), 20 + N)
    got = _run_gemm(ctx, cc.CC_BM1, A, M, Lt, N, S, 5, (Lt, S, N, N, N))
    want = values.bm1(A, M)
    err = float(np.max(np.abs(got - want) / np.abs(want)))
    assert err <= 1e-10, err


@pytest.mark.parametrize("Lt,N,S", [(2, 8, 4), (1, 12, 64), (2, 16, 64), (1, 24, 64), (1, 33, 8), (2, 20, 3)])
def test_bb2_ozaki_split_k(ctx, Lt, N, S):
    """BB2 (K = S N^2 up to 36864 complex terms: 1..5 split-K chunks of 8192, FP64 partials
    summed in chunk order) vs the oracle's BB2; bit-identical on a repeat (deterministic)."""
    from paper_2511_02257_b200 import cc
    A = _phase_limited((Lt, S, N, N, N), 30 + N)
    B = _phase_limited((Lt, S, N, N, N), 40 + N)
    got = _run_gemm(ctx, cc.CC_BB2, A, B, Lt, N, S, 5, (Lt, N, N))
    want = values.bb2(A, B)
    err = float(np.max(np.abs(got - want) / np.abs(want)))
    assert err <= 1e-10, err
    again = _run_gemm(ctx, cc.CC_BB2, A, B, Lt, N, S, 5, (Lt, N, N))
    assert np.array_equal(got, again)


def test_gemm_ozaki_time_batches(ctx):
    """A workspace that holds one time slice only: the engine runs the problem slice by slice,
    same values as with the full workspace."""
    from paper_2511_02257_b200 import cc
    Lt, N, S = 4, 16, 8
    A = _phase_limited((Lt, S, N, N, N), 51)
    B = _phase_limited((Lt, S, N, N, N), 52)
    one = cc.cc_gemm_ozaki_workspace_bytes(cc.CC_BB2, 1, N, S, 5)
    got = _run_gemm(ctx, cc.CC_BB2, A, B, Lt, N, S, 5, (Lt, N, N), ws_bytes=one)
    full = _run_gemm(ctx, cc.CC_BB2, A, B, Lt, N, S, 5, (Lt, N, N))
    assert np.array_equal(got, full)


def test_executor_ozaki_baryon_dags():
    """c3 (nucleon) and c4 (two-baryon, capped pool with evictions) DAGs with every GEMM kind
    on the Ozaki engine (flags bit 6): roots and correlators within 1e-10 of the oracle."""
    from synth import dags
    from oracle.dag import Dag
    from oracle import lru, tree
    from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close
    w = dags.config_c3(N=12, Lt=2, S=64)
    dag = Dag(w)
    _, roots, corr, st, ex = run_gpu(w, flags=64, arena_mb=1024)
    r_or, c_or = values.run_workload(w, dag)
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)
    w = dags.config_c4(N=8, Lt=1, S=4, n_trees=120, n_corr=4)
    dag = Dag(w)
    cap = 7 * 16 * 4 * 8 ** 3
    for nu in (False, True):
        _, roots, corr, st, ex = run_gpu(w, cap=cap, flags=64, evict_next_use=nu)
        p = lru.plan(dag, tree.schedule(dag), cap, policy="next_use" if nu else "lru")
        assert ex["h2d_bytes"] == p["h2d_bytes"] and ex["d2h_bytes"] == p["d2h_bytes"]
        r_or, c_or = values.run_workload(w, dag)
        assert_roots_close(roots, r_or)
        assert_corr_close(dag, r_or, corr, c_or)


def test_executor_auto_flag():
    """CC_EXEC_AUTO (flags bit 7): a c2-shaped DAG at N=72 stays on the dataflow worker (one
    persistent launch + correlator), a c5-shaped one at N=512 goes to the Ozaki engine (N = 256
    stays on the worker since the round-2 measurements); all match the oracle."""
    from synth import dags
    from oracle.dag import Dag
    from paper_2511_02257_b200 import cc
    from gpu_helpers import run_gpu, assert_roots_close
    w = dags.config_c2(N=72, Lt=3, n_loop4=40, n_loop2=4, n_corr=3)
    _, roots, _, _, ex = run_gpu(w, flags=cc.EXEC_AUTO)
    assert ex["n_kernels"] <= 3
    assert_roots_close(roots, values.run_workload(w, Dag(w))[0])
    w = dags.config_c5(N=256, Lt=2, n_pairs=12, n_trees=30, n_corr=3)
    _, roots, _, _, ex = run_gpu(w, flags=cc.EXEC_AUTO, arena_mb=2048)
    assert ex["n_kernels"] <= 3
    assert_roots_close(roots, values.run_workload(w, Dag(w))[0])
    w = dags.config_c5(N=512, Lt=2, n_pairs=12, n_trees=30, n_corr=3)
    _, roots, _, _, ex = run_gpu(w, flags=cc.EXEC_AUTO, arena_mb=3072)
    assert ex["n_kernels"] > 10
    assert_roots_close(roots, values.run_workload(w, Dag(w))[0])


def test_bb2_ozaki_random_phase_scale(ctx):
    """BB2 with random-phase data (terms of both signs, cancellation) across 2 split-K chunks:
    within 1e-10 of the |A||B| error scale (V-4), like the FP64 DMMA path."""
    from paper_2511_02257_b200 import cc
    Lt, N, S = 1, 16, 64
    A = _random_phase((Lt, S, N, N, N), 61)
    B = _random_phase((Lt, S, N, N, N), 62)
    got = _run_gemm(ctx, cc.CC_BB2, A, B, Lt, N, S, 5, (Lt, N, N))
    want = values.bb2(A, B)
    scale = sum(np.matmul(np.abs(A[:, s]).reshape(Lt, N, N * N), np.abs(B[:, s]).reshape(Lt, N * N, N))
                for s in range(S))
    assert np.all(np.abs(got - want) <= 1e-10 * scale)
