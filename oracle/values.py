"""O7 — values: the four contraction kinds and the correlator sums, in complex128.

TEST INFRASTRUCTURE (see oracle/__init__.py).

The paper names the operations but never writes their indices (reading V-1,
DESIGN.md): "exterior contract" for interior nodes and "contract all" for roots
(P:867), complexity classes O(N^3)/O(N^4), 64 spin components
(P:59).  Definitions used (each written out with one library matmul as a step):
  MM1(A,B)[t,i,k]     = sum_j A[t,i,j] B[t,j,k]                  (MxM, O(N^3))
  BM1(A,M)[t,s,i,j,l] = sum_k A[t,s,i,j,k] M[t,k,l]              (BxM, O(N^4))
  BB2(A,B)[t,i,l]     = sum_s sum_{j,k} A[t,s,i,j,k] B[t,s,j,k,l] (BxB, O(N^4))
  TR_MM(A,B)[t]       = sum_{i,j} A[t,i,j] B[t,j,i]              (contract all)
Correlator (reading V-2): C_c[t] = sum over terms (c, T, coef) of coef * root_T[t],
summed in term input order.
BxBxB kinds (tritium class, Table II O(N^5) P:813; size classes P:871-872; readings T4-1..T4-4):
  BB1(A,B)[t,i,j,l,m] = sum_s sum_k A[t,s,i,j,k] B[t,s,k,l,m]      (baryon x baryon -> tetra)
  BT2(A,X)[t,s,m,i,j] = sum_{k,l} A[t,s,m,k,l] X[t,k,l,i,j]        (baryon x tetra -> baryon)
  BB3(A,B)[t]         = sum_s sum_{i,j,k} A[t,s,i,j,k] B[t,s,k,j,i] (baryon x baryon contract all)
Precision: complex128 throughout (P:59 pins 16 B per element; reading V-3).
"""
import numpy as np

from synth import rng as srng
from synth.dags import LEAF_M, LEAF_B, MM1, BM1, BB2, TR_MM, BB1, BT2, BB3


def mm1(A, B):
    return np.matmul(A, B)


def bm1(A, M):
    Lt, S, N = A.shape[0], A.shape[1], A.shape[2]
    C = np.matmul(A.reshape(Lt, S * N * N, N), M)
    return C.reshape(A.shape)


def bb2(A, B):
    Lt, S, N = A.shape[0], A.shape[1], A.shape[2]
    C = np.zeros((Lt, N, N), dtype=np.complex128)
    for s in range(S):                       # sum over the spin index s
        C += np.matmul(A[:, s].reshape(Lt, N, N * N), B[:, s].reshape(Lt, N * N, N))
    return C


def tr_mm(A, B):
    return (A * np.swapaxes(B, 1, 2)).sum(axis=(1, 2))


def bb1(A, B):
    Lt, S, N = A.shape[0], A.shape[1], A.shape[2]
    T = np.zeros((Lt, N * N, N * N), dtype=np.complex128)
    for s in range(S):                       # sum over the spin index s
        T += np.matmul(A[:, s].reshape(Lt, N * N, N), B[:, s].reshape(Lt, N, N * N))
    return T.reshape(Lt, N, N, N, N)


def bt2(A, X):
    Lt, S, N = A.shape[0], A.shape[1], A.shape[2]
    C = np.matmul(A.reshape(Lt, S * N, N * N), X.reshape(Lt, N * N, N * N))
    return C.reshape(Lt, S, N, N, N)


def bb3(A, B):
    return (A * np.transpose(B, (0, 1, 4, 3, 2))).sum(axis=(1, 2, 3, 4))


KERNELS = {MM1: mm1, BM1: bm1, BB2: bb2, TR_MM: tr_mm, BB1: bb1, BT2: bt2, BB3: bb3}


def leaf_shape(op, Lt, N, S):
    return (Lt, N, N) if op == LEAF_M else (Lt, S, N, N, N)


def synthetic_leaf(w, leaf_id, op, t_range=None):
    """The leaf tensor of workload w, from the shared generator (synth.rng)."""
    shape = leaf_shape(op, w.Lt, w.N, w.S)
    sigma = srng.meson_sigma(w.N) if op == LEAF_M else srng.baryon_sigma(w.N, w.S)
    return srng.leaf_tensor(w.data_seed, leaf_id, shape, sigma, w.leaf_mode, t_range)


def evaluate(dag, leaf, roots_only=True):
    """Evaluate every node needed by the trees.  `leaf(id)` returns a leaf tensor.
    Returns {tree_id: root value [Lt']} (and all node values if roots_only=False).
    Intermediates are dropped once their last parent has been evaluated."""
    nodes = dag.nodes
    val = {}
    left = {u: len(n.parents) for u, n in nodes.items()}
    keep = {}
    for u in dag.topo:
        n = nodes[u]
        if not n.child:
            val[u] = leaf(u)
            continue
        a, b = n.child
        val[u] = KERNELS[n.op](val[a], val[b])
        for c in n.child:
            left[c] -= 1
            if left[c] == 0 and roots_only:
                del val[c]
    roots = {t: val[dag.trees[t][0]] for t in dag.tree_ids}
    if not roots_only:
        keep = val
    return roots if roots_only else (roots, keep)


def correlators(dag, roots):
    """C_c[t] = sum_{(c,T,coef)} coef * root_T[t], terms in input order."""
    out = {}
    for (c, t, coef) in dag.terms:
        if c not in out:
            out[c] = np.zeros_like(roots[t])
        out[c] = out[c] + coef * roots[t]
    return out


def term_scale(dag, roots):
    """sum_terms |coef * root| per correlator (the V-4 tolerance scale)."""
    out = {}
    for (c, t, coef) in dag.terms:
        out[c] = out.get(c, 0.0) + np.abs(coef * roots[t])
    return out


def run_workload(w, dag=None, t_range=None):
    """Roots and correlators of a synth Workload (optionally time slices t_range only)."""
    from .dag import Dag
    dag = dag or Dag(w)
    ops = {u: n.op for u, n in dag.nodes.items()}
    roots = evaluate(dag, lambda u: synthetic_leaf(w, u, ops[u], t_range))
    return roots, correlators(dag, roots)
