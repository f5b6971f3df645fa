"""Pins of oracle O7 (values) against closed forms, brute-force loops and invariants.

Definitions: DESIGN reading V-1 (index semantics of MM1/BM1/BB2/TR_MM; P:120,
P:806-813), correlator = sum of terms (reading V-2).
- brute force: plain Python index loops on tiny tensors (not the numpy path)
- closed forms: all-ones J (MM1 = N J, TR = N^2, c1 loop = N^4), identity, rank-1
  dyadic leaves (trace of a product of rank-1 matrices factorises), spin-separable
  baryons (BM1/BB2 factorise into scalars)
- invariants: trace cyclicity, linearity, per-time-slice independence
- the shared generator: phase bound of the phase-limited mode, determinism
"""
import itertools

import numpy as np
import pytest

from synth import dags, rng as srng
from oracle import values
from oracle.dag import Dag


def _rand(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


def test_brute_force_loops_tiny():
    Lt, N, S = 2, 3, 2
    A = _rand((Lt, N, N), 1)
    B = _rand((Lt, N, N), 2)
    Ab = _rand((Lt, S, N, N, N), 3)
    Bb = _rand((Lt, S, N, N, N), 4)
    R = range(N)
    mm = np.zeros((Lt, N, N), complex)
    tr = np.zeros(Lt, complex)
    bm = np.zeros((Lt, S, N, N, N), complex)
    bb = np.zeros((Lt, N, N), complex)
    for t in range(Lt):
        for i, k in itertools.product(R, R):
            mm[t, i, k] = sum(A[t, i, j] * B[t, j, k] for j in R)
        tr[t] = sum(A[t, i, j] * B[t, j, i] for i in R for j in R)
        for s, i, j, l in itertools.product(range(S), R, R, R):
            bm[t, s, i, j, l] = sum(Ab[t, s, i, j, k] * A[t, k, l] for k in R)
        for i, l in itertools.product(R, R):
            bb[t, i, l] = sum(Ab[t, s, i, j, k] * Bb[t, s, j, k, l]
                              for s in range(S) for j in R for k in R)
    np.testing.assert_allclose(values.mm1(A, B), mm, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(values.tr_mm(A, B), tr, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(values.bm1(Ab, A), bm, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(values.bb2(Ab, Bb), bb, rtol=1e-13, atol=1e-13)


def test_all_ones_closed_forms():
    Lt, N = 4, 32
    J = np.ones((Lt, N, N), complex)
    assert np.array_equal(values.mm1(J, J), N * J)
    assert np.array_equal(values.tr_mm(J, J), np.full(Lt, N * N, complex))
    # c1 with all-ones leaves: TR(MM1(J,J), MM1(J,J)) = N^4 exactly (2^20 at N=32)
    w = dags.config_c1(N=N, Lt=Lt)
    dag = Dag(w)
    roots = values.evaluate(dag, lambda u: J)
    assert np.array_equal(roots[0], np.full(Lt, float(N) ** 4, complex))


def test_bxbxb_brute_force_loops_tiny():
    """BB1 / BT2 / BB3 (readings T4-1..T4-3) against plain index loops over every index."""
    Lt, N, S = 2, 3, 2
    A = _rand((Lt, S, N, N, N), 11)
    B = _rand((Lt, S, N, N, N), 12)
    X = _rand((Lt, N, N, N, N), 13)
    R = range(N)
    bb1 = np.zeros((Lt, N, N, N, N), complex)
    bt2 = np.zeros((Lt, S, N, N, N), complex)
    bb3 = np.zeros(Lt, complex)
    for t in range(Lt):
        for i, j, l, m in itertools.product(R, R, R, R):
            bb1[t, i, j, l, m] = sum(A[t, s, i, j, k] * B[t, s, k, l, m] for s in range(S) for k in R)
        for s, m, i, j in itertools.product(range(S), R, R, R):
            bt2[t, s, m, i, j] = sum(A[t, s, m, k, l] * X[t, k, l, i, j] for k in R for l in R)
        bb3[t] = sum(A[t, s, i, j, k] * B[t, s, k, j, i] for s in range(S) for i in R for j in R for k in R)
    np.testing.assert_allclose(values.bb1(A, B), bb1, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(values.bt2(A, X), bt2, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(values.bb3(A, B), bb3, rtol=1e-13, atol=1e-13)
    # numpy.einsum as a third opinion
    np.testing.assert_allclose(np.einsum("tsijk,tsklm->tijlm", A, B), bb1, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(np.einsum("tsmkl,tklij->tsmij", A, X), bt2, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(np.einsum("tsijk,tskji->t", A, B), bb3, rtol=1e-13, atol=1e-13)


def test_bxbxb_closed_forms():
    """All-ones baryons J_B and tetra J_T: BB1(J_B, J_B) = S N J_T (sum over s, k), BT2(J_B, J_T)
    = N^2 J_B (sum over k, l), BB3(J_B, J_B) = S N^3; a tritium-family tree of all-ones leaves
    (c6 family A: BB3(BT2(J, BB1(BT2(J, BB1(J, J)), J)), J)) is then exactly
    S N^3 (S N N^2)^2 = S^3 N^9; spin-separable baryons A = sa (x) a, B = sb (x) b factorise."""
    Lt, N, S = 2, 4, 3
    JB = np.ones((Lt, S, N, N, N), complex)
    JT = np.ones((Lt, N, N, N, N), complex)
    assert np.array_equal(values.bb1(JB, JB), S * N * JT)
    assert np.array_equal(values.bt2(JB, JT), N * N * JB)
    assert np.array_equal(values.bb3(JB, JB), np.full(Lt, S * N ** 3, complex))
    w = dags.config_c6(N=N, Lt=Lt, S=S, n_trees=12, p_meson=0.0)
    dag = Dag(w)
    roots = values.evaluate(dag, lambda u: JB)
    for t in dag.tree_ids:
        np.testing.assert_array_equal(roots[t], np.full(Lt, float(S ** 3 * N ** 9), complex))
    sa, sb = _rand((Lt, S), 21), _rand((Lt, S), 22)
    a, b = _rand((Lt, N, N, N), 23), _rand((Lt, N, N, N), 24)
    X = _rand((Lt, N, N, N, N), 25)
    A = np.einsum("ts,tijk->tsijk", sa, a)
    B = np.einsum("ts,tijk->tsijk", sb, b)
    ss = np.einsum("ts,ts->t", sa, sb)
    np.testing.assert_allclose(values.bb1(A, B), ss[:, None, None, None, None] * np.einsum("tijk,tklm->tijlm", a, b),
                               rtol=1e-12)
    np.testing.assert_allclose(values.bb3(A, B), ss * np.einsum("tijk,tkji->t", a, b), rtol=1e-12)
    np.testing.assert_allclose(values.bt2(A, X), np.einsum("ts,tmij->tsmij", sa, np.einsum("tmkl,tklij->tmij", a, X)),
                               rtol=1e-12)


def test_identity_and_transpose_structure():
    Lt, N = 2, 5
    I = np.broadcast_to(np.eye(N, dtype=complex), (Lt, N, N))
    A = _rand((Lt, N, N), 7)
    np.testing.assert_array_equal(values.mm1(I, A), A)
    np.testing.assert_array_equal(values.mm1(A, I), A)
    assert np.array_equal(values.tr_mm(I, I), np.full(Lt, N, complex))
    # TR_MM(A, B) = trace(A B); with B = I it is trace(A) = sum of the diagonal
    np.testing.assert_allclose(values.tr_mm(A, I), np.einsum("tii->t", A), rtol=1e-14)


def test_rank1_dyadic_product_trace_exact():
    """Tr(M1 M2 M3 M4) with Mx = u_x v_x^T equals (v1.u2)(v2.u3)(v3.u4)(v4.u1);
    dyadic-rational entries make every partial sum exact in FP64."""
    r = np.random.default_rng(5)
    Lt, N = 3, 16
    u = [(r.integers(-8, 9, (Lt, N)) + 1j * r.integers(-8, 9, (Lt, N))) / 8 for _ in range(4)]
    v = [(r.integers(-8, 9, (Lt, N)) + 1j * r.integers(-8, 9, (Lt, N))) / 8 for _ in range(4)]
    M = [np.einsum("ti,tj->tij", u[x], v[x]) for x in range(4)]
    X = values.mm1(M[0], M[1])
    Y = values.mm1(M[2], M[3])
    got = values.tr_mm(X, Y)
    dot = lambda a, b: (a * b).sum(axis=1)  # noqa: E731
    want = dot(v[0], u[1]) * dot(v[1], u[2]) * dot(v[2], u[3]) * dot(v[3], u[0])
    assert np.array_equal(got, want)


def test_spin_separable_baryons():
    """B[t,s,i,j,k] = sigma_s * b[i,j,k]: BB2(A,B) = (sum_s a_s b_s) * sum_{jk} a[i,j,k] b[j,k,l];
    BM1 keeps the spin factor."""
    r = np.random.default_rng(9)
    Lt, S, N = 2, 4, 3
    sa, sb = _rand((Lt, S), 1), _rand((Lt, S), 2)
    a, b = _rand((Lt, N, N, N), 3), _rand((Lt, N, N, N), 4)
    A = np.einsum("ts,tijk->tsijk", sa, a)
    B = np.einsum("ts,tijk->tsijk", sb, b)
    want = np.einsum("ts,ts->t", sa, sb)[:, None, None] * np.einsum("tijk,tjkl->til", a, b)
    np.testing.assert_allclose(values.bb2(A, B), want, rtol=1e-12)
    M = _rand((Lt, N, N), 5)
    want_bm = np.einsum("ts,tijl->tsijl", sa, np.einsum("tijk,tkl->tijl", a, M))
    np.testing.assert_allclose(values.bm1(A, M), want_bm, rtol=1e-12)


def test_trace_cyclicity_and_linearity():
    Lt, N = 2, 8
    M = [_rand((Lt, N, N), s) for s in range(4)]
    r1 = values.tr_mm(values.mm1(M[0], M[1]), values.mm1(M[2], M[3]))
    r2 = values.tr_mm(values.mm1(M[1], M[2]), values.mm1(M[3], M[0]))
    np.testing.assert_allclose(r1, r2, rtol=1e-12)
    c = 0.3 - 1.7j
    np.testing.assert_allclose(values.mm1(c * M[0] + M[1], M[2]),
                               c * values.mm1(M[0], M[2]) + values.mm1(M[1], M[2]), rtol=1e-12)


def test_time_slices_independent():
    w = dags.config_c2(N=6, Lt=4, n_loop4=20, n_loop2=3)
    roots_full, corr_full = values.run_workload(w)
    roots_part, corr_part = values.run_workload(w, t_range=(1, 3))
    for t in roots_full:
        np.testing.assert_array_equal(roots_full[t][1:3], roots_part[t])


def test_correlator_sum_of_terms():
    w = dags.fixture_dstar()
    w2 = dags.config_c2(N=4, Lt=2, n_loop4=10, n_loop2=2, n_corr=3)
    dag = Dag(w2)
    roots, corr = values.run_workload(w2, dag)
    for c in corr:
        want = sum(coef * roots[t] for (cc, t, coef) in dag.terms if cc == c)
        np.testing.assert_allclose(corr[c], want, rtol=1e-15)


def scaled_ones_scalars(w):
    """Closed form for leaves c_u * J (J the all-ones matrix, c_u = scaled_ones_factor(u)):
    MM1(xJ, yJ) = x y N J and TR_MM(xJ, yJ) = x y N^2 (sum of N^2 equal entries), so every node
    is (scalar) * J and every root an integer; returns {node: scalar} in Python integers."""
    nodes = {n[0]: n for n in w.nodes}
    memo = {}

    def sc(u):
        if u not in memo:
            (_, op, a, b, _) = nodes[u]
            if op == dags.LEAF_M:
                memo[u] = scaled_ones_factor(u)
            elif op == dags.MM1:
                memo[u] = sc(a) * sc(b) * w.N
            elif op == dags.TR_MM:
                memo[u] = sc(a) * sc(b) * w.N * w.N
            else:
                raise ValueError(op)
        return memo[u]
    return {u: sc(u) for u in nodes}


def scaled_ones_factor(u):
    return (u % 5) - 2 or 3          # small nonzero integers of both signs


def test_correlator_closed_form_scaled_ones():
    """Pins values.correlators (and the MM1 / TR_MM chain) against exact integers: with leaves
    c_u J every root is an integer (scaled_ones_scalars) and, with Gaussian-integer coefficients,
    every correlator entry C_c[t] = sum over c's terms of coef * root is an exact Gaussian integer
    (P:54), summed here in Python integers from the DAG structure alone."""
    N, Lt = 6, 3
    w = dags.config_c2(N=N, Lt=Lt, n_loop4=40, n_loop2=5, n_corr=4, coefs="complex")
    assert any(im != 0 for (_, _, _, im) in w.terms)
    dag = Dag(w)
    sc = scaled_ones_scalars(w)
    roots = values.evaluate(dag, lambda u: scaled_ones_factor(u) * np.ones((Lt, N, N), complex))
    corr = values.correlators(dag, roots)
    root_of = dict(w.trees)
    want = {}
    for (c, t, re, im) in w.terms:
        r = sc[root_of[t]]
        pre, pim = want.get(c, (0, 0))
        want[c] = (pre + int(re) * r, pim + int(im) * r)
    assert set(corr) == set(want)
    for c, (re, im) in want.items():
        np.testing.assert_array_equal(corr[c], np.full(Lt, complex(re, im)))
    for t, r in root_of.items():
        np.testing.assert_array_equal(roots[t], np.full(Lt, complex(sc[r], 0)))


def test_generator_phase_bound_and_determinism():
    v = srng.leaf_values(1, 7, 0, 4096, 0.5, srng.MODE_PHASE_LIMITED)
    assert np.all(np.abs(np.angle(v)) <= np.arctan(0.125 / 0.75) + 1e-15)
    assert np.all((v.real >= 0.375) & (v.real < 0.625))
    v2 = srng.leaf_values(1, 7, 1000, 100, 0.5)
    np.testing.assert_array_equal(v[1000:1100], v2)
    assert not np.array_equal(srng.leaf_values(2, 7, 0, 8, 0.5), v[:8])
    # splitmix64 reference value: splitmix64 of state 0 (first output of seed 0) is
    # 0xE220A8397B1DCDAF (the published SplitMix64 test vector)
    assert int(srng.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
