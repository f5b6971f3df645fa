"""Degenerate and edge cases of the CUDA path (through the C ABI) against the oracle:
N = 1 (scalar mesons), all-zero leaves (exact zeros on both engines), a TIME part with no
time slices (rejected) next to one with a single slice, and a DAG of only two-meson traces."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import dags  # noqa: E402
from oracle import values  # noqa: E402
from oracle.dag import Dag  # noqa: E402
from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close  # noqa: E402


@pytest.mark.parametrize("flags", [0, 16, 64])
def test_scalar_mesons_N1(flags):
    """N = 1: every contraction is a product of complex scalars per time slice."""
    w = dags.config_c2(N=1, Lt=3, n_loop4=12, n_loop2=3, n_corr=2)
    dag = Dag(w)
    _, roots, corr, _, _ = run_gpu(w, flags=flags)
    r_or, c_or = values.run_workload(w, dag)
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, c_or)


@pytest.mark.parametrize("flags", [0, 64])
def test_all_zero_leaves_give_exact_zeros(flags):
    w = dags.config_c2(N=40, Lt=2, n_loop4=20, n_loop2=2, n_corr=2)
    shape = {dags.LEAF_M: (w.Lt, w.N, w.N)}
    _, roots, corr, _, _ = run_gpu(w, flags=flags, leaf_fn=lambda u, op: np.zeros(shape[op], dtype=np.complex128))
    assert all(np.array_equal(r, np.zeros_like(r)) for r in roots.values())
    assert all(np.array_equal(c, np.zeros_like(c)) for c in corr.values())


def test_empty_time_part_is_rejected():
    """Four TIME parts of Lt = 2: part 0 owns no slice, which cc_partition rejects with
    CC_E_INVAL (documented); part 3 owns slice 1 and matches the oracle there."""
    from paper_2511_02257_b200 import cc
    w = dags.config_c2(N=16, Lt=2, n_loop4=10, n_loop2=2, n_corr=2)
    with pytest.raises(cc.CCError) as ei:
        run_gpu(w, part=(4, 0, cc.PART_TIME))
    assert ei.value.code == "INVAL"
    dag = Dag(w)
    _, roots, _, _, _ = run_gpu(w, part=(4, 3, cc.PART_TIME))
    r_or, _ = values.run_workload(w, dag, t_range=(1, 2))
    assert_roots_close({k: roots[k] for k in r_or}, r_or)


def test_traces_only_dag():
    """A DAG whose every tree is TR_MM(leaf, leaf): no GEMM work at all."""
    w = dags.config_c2(N=48, Lt=3, n_loop4=0, n_loop2=8, n_corr=3)
    dag = Dag(w)
    for flags in (0, 1, 16):
        _, roots, corr, _, _ = run_gpu(w, flags=flags)
        r_or, c_or = values.run_workload(w, dag)
        assert_roots_close(roots, r_or)
        assert_corr_close(dag, r_or, corr, c_or)
