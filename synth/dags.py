"""Seeded synthetic contraction-DAG workloads (structure only; no method arithmetic).

A workload is the input of the paper's problem statement (§II-B,
lines 151-183): k rooted contraction trees over shared hadron nodes, merged
into one DAG, plus the correlator terms that sum tree roots.
Both the oracle and the CUDA path consume the same `Workload` object; neither
derives anything from the other.

Op codes mirror include/cc.h (`cc_op`).  Index semantics of the typed ops are
DESIGN.md reading V-1:
  MM1(A,B)[t,i,k]     = sum_j A[t,i,j] B[t,j,k]                 meson x meson
  BM1(A,M)[t,s,i,j,l] = sum_k A[t,s,i,j,k] M[t,k,l]             baryon x meson
  BB2(A,B)[t,i,l]     = sum_s sum_{j,k} A[t,s,i,j,k] B[t,s,j,k,l] baryon x baryon
  TR_MM(A,B)[t]       = sum_{i,j} A[t,i,j] B[t,j,i]              contract-all (root)
BxBxB kinds (tritium class, readings T4-1..T4-4):
  BB1(A,B)[t,i,j,l,m] = sum_s sum_k A[t,s,i,j,k] B[t,s,k,l,m]    baryon x baryon -> tetra
  BT2(A,X)[t,s,m,i,j] = sum_{k,l} A[t,s,m,k,l] X[t,k,l,i,j]      baryon x tetra -> baryon
  BB3(A,B)[t]         = sum_s sum_{i,j,k} A[t,s,i,j,k] B[t,s,k,j,i]  contract-all (root)
LEAF_X / OP_X are abstract nodes with explicit sizes (scheduling-only DAGs,
e.g. the Table I example); they carry no tensor semantics.

Recipes of the five BASELINE.json configs are DESIGN.md §"Input recipe".
"""
from dataclasses import dataclass, field
import numpy as np

LEAF_M, LEAF_B, MM1, BM1, BB2, TR_MM, LEAF_X, OP_X, BB1, BT2, BB3 = range(11)
OP_NAMES = ["leafM", "leafB", "MM1", "BM1", "BB2", "TR_MM", "leafX", "OPX", "BB1", "BT2", "BB3"]
N_OPS = len(OP_NAMES)
LEAF_OPS = (LEAF_M, LEAF_B, LEAF_X)


@dataclass
class Workload:
    name: str
    Lt: int
    N: int
    S: int
    nodes: list = field(default_factory=list)   # (id, op, a, b, size) ; size 0 = from shape
    trees: list = field(default_factory=list)   # (tree_id, root_id)
    terms: list = field(default_factory=list)   # (corr_id, tree_id, re, im)
    data_seed: int = 1
    leaf_mode: int = 0                          # synth.rng MODE_*

    def leaf_ids(self):
        return [n[0] for n in self.nodes if n[1] in LEAF_OPS]

    def node_map(self):
        return {n[0]: n for n in self.nodes}

    def to_text(self):
        """Text format of include/cc.h (cc_load_dag_file)."""
        out = ["# %s" % self.name, "dims %d %d %d" % (self.Lt, self.N, self.S)]
        for (i, op, a, b, size) in self.nodes:
            if op in LEAF_OPS:
                s = "node %d %s" % (i, OP_NAMES[op])
            else:
                s = "node %d %s %d %d" % (i, OP_NAMES[op], a, b)
            if size:
                s += " size %d" % size
            out.append(s)
        for (t, r) in self.trees:
            out.append("tree %d %d" % (t, r))
        for (c, t, re, im) in self.terms:
            out.append("term %d %d %r %r" % (c, t, float(re), float(im)))
        return "\n".join(out) + "\n"


class Builder:
    def __init__(self, name, Lt, N, S):
        self.w = Workload(name, Lt, N, S)
        self._next = 0
        self._dedupe = {}

    def leaf(self, op, size=0):
        i = self._next
        self._next += 1
        self.w.nodes.append((i, op, -1, -1, size))
        return i

    def op(self, op, a, b, size=0, share=True):
        key = (op, a, b)
        if share and key in self._dedupe:
            return self._dedupe[key]
        i = self._next
        self._next += 1
        self.w.nodes.append((i, op, a, b, size))
        if share:
            self._dedupe[key] = i
        return i

    def tree(self, root):
        t = len(self.w.trees)
        self.w.trees.append((t, root))
        return t

    def term(self, corr, tree, re=1.0, im=0.0):
        self.w.terms.append((corr, tree, re, im))


# ----------------------------------------------------------------------------
# Fixtures
# ----------------------------------------------------------------------------

def fixture_dstar():
    """D* (SURVEY §8(c) G-1): the DAG that reproduces every size of PAPER.md
    Table I (l.219-246).  Leaves a,b,c,d; e=(b,c), f=(a,b), g=(a,e), h=(d,e);
    trees T0={f,a,b}, T1={g,a,e,b,c}, T2={h,d,e,b,c}; unit sizes.
    Ids: a=0 b=1 c=2 d=3 e=4 f=5 g=6 h=7 (alphabetical)."""
    w = Workload("Dstar", 1, 1, 1)
    for i in range(4):
        w.nodes.append((i, LEAF_X, -1, -1, 1))
    w.nodes += [(4, OP_X, 1, 2, 1), (5, OP_X, 0, 1, 1), (6, OP_X, 0, 4, 1), (7, OP_X, 3, 4, 1)]
    w.trees = [(0, 5), (1, 6), (2, 7)]
    w.terms = [(0, 0, 1.0, 0.0), (0, 1, 1.0, 0.0), (0, 2, 1.0, 0.0)]
    return w


def fixture_next_use():
    """Eviction-policy fixture (reading E-9): leaves a,b,c,d; roots (one tree each)
    s1=(a,b), s2=(c,a), s3=(d,b), s4=(c,d), s5=(b,a); unit sizes; replayed in id order.
    Ids: a=0 b=1 c=2 d=3 s1=4 .. s5=8."""
    w = Workload("NextUse", 1, 1, 1)
    for i in range(4):
        w.nodes.append((i, LEAF_X, -1, -1, 1))
    w.nodes += [(4, OP_X, 0, 1, 1), (5, OP_X, 2, 0, 1), (6, OP_X, 3, 1, 1), (7, OP_X, 2, 3, 1), (8, OP_X, 1, 0, 1)]
    w.trees = [(k, 4 + k) for k in range(5)]
    w.terms = [(0, k, 1.0, 0.0) for k in range(5)]
    return w


def fixture_f1():
    """SPEC.md fixture F1: leaves a,b,l; e=(b,l); g=(e,a); h=(e,a);
    f=(a,b); T0=g-tree, T1=h-tree, T2=f-tree; unit sizes.
    Ids (alphabetical): a=0 b=1 e=2 f=3 g=4 h=5 l=6."""
    w = Workload("F1", 1, 1, 1)
    w.nodes = [(0, LEAF_X, -1, -1, 1), (1, LEAF_X, -1, -1, 1), (6, LEAF_X, -1, -1, 1),
               (2, OP_X, 1, 6, 1), (4, OP_X, 2, 0, 1), (5, OP_X, 2, 0, 1), (3, OP_X, 0, 1, 1)]
    w.trees = [(0, 4), (1, 5), (2, 3)]
    w.terms = [(0, 0, 1.0, 0.0), (0, 1, 1.0, 0.0), (0, 2, 1.0, 0.0)]
    return w


# ----------------------------------------------------------------------------
# Random DAGs for the scheduler/planner property tests
# ----------------------------------------------------------------------------

def random_dag(seed, n_leaves=6, n_trees=4, max_ops_per_tree=4, share_p=0.5,
               typed=False, max_size=4, Lt=2, N=4, S=2):
    """Random binary contraction DAG built tree by tree.

    Each tree combines operands drawn from the shared leaf pool or from interior
    nodes of earlier trees (probability share_p) into a binary tree; identical
    (op, a, b) contractions are merged, which is how DAG sharing arises.
    typed=False: abstract nodes with random sizes in [1, max_size].
    typed=True : meson-only DAG (leafM, MM1 interiors, TR_MM roots) with real shapes.
    Trees are closed under operands by construction (tree = closure of its root).
    """
    rng = np.random.default_rng(seed)
    b = Builder("random%d" % seed, Lt, N, S)
    lop = LEAF_M if typed else LEAF_X
    iop = MM1 if typed else OP_X
    rop = TR_MM if typed else OP_X

    def sz():
        return 0 if typed else int(rng.integers(1, max_size + 1))

    leaves = [b.leaf(lop, sz()) for _ in range(n_leaves)]
    interiors = []
    for _ in range(n_trees):
        n_ops = int(rng.integers(1, max_ops_per_tree + 1))
        # operands: n_ops + 1 of them, combined pairwise n_ops times (last = root)
        operands = []
        for _ in range(n_ops + 1):
            if interiors and rng.random() < share_p:
                operands.append(interiors[int(rng.integers(len(interiors)))])
            else:
                operands.append(leaves[int(rng.integers(len(leaves)))])
        # make operands distinct where possible; a == b is not a legal contraction
        while len(operands) > 1:
            i = int(rng.integers(len(operands) - 1))
            x, y = operands[i], operands[i + 1]
            if len(operands) == 2:
                if x == y:
                    y = next(l for l in leaves if l != x)
                root = b.op(rop, x, y, sz(), share=False)
                operands = [root]
                break
            if x == y:
                y = next(l for l in leaves if l != x)
            v = b.op(iop, x, y, sz())
            if v not in interiors:
                interiors.append(v)
            operands[i:i + 2] = [v]
        if len(operands) == 1 and operands[0] in leaves:
            # n_ops + 1 == 1 cannot happen (n_ops >= 1); guard anyway
            continue
        t = b.tree(operands[0])
        b.term(int(rng.integers(3)), t, float(rng.choice([1.0, -1.0])), 0.0)
    _prune(b.w)
    return b.w


def _prune(w):
    """Drop nodes no tree references (an unreferenced leaf would be isolated)."""
    used = set()
    for (i, op, a, bb, s) in w.nodes:
        if op not in LEAF_OPS:
            used.update((a, bb))
    roots = {r for (_, r) in w.trees}
    w.nodes = [n for n in w.nodes if n[0] in used or n[0] in roots]


# ----------------------------------------------------------------------------
# The five BASELINE.json configs (structure); DESIGN.md §"Input recipe"
# ----------------------------------------------------------------------------

def config_c1(N=32, Lt=4):
    """c1: single pi-pi correlator, 1 graph: root = TR_MM(MM1(M0,M1), MM1(M2,M3))."""
    b = Builder("c1_pipi_N%d_Lt%d" % (N, Lt), Lt, N, 1)
    m = [b.leaf(LEAF_M) for _ in range(4)]
    x = b.op(MM1, m[0], m[1])
    y = b.op(MM1, m[2], m[3])
    t = b.tree(b.op(TR_MM, x, y, share=False))
    b.term(0, t)
    return b.w


# Gaussian-integer term coefficients (coefs="complex"): exact in FP64, both signs, both parts
COMPLEX_COEFS = [(1.0, 2.0), (-1.0, 1.0), (2.0, -1.0), (0.0, -3.0), (-2.0, 0.0), (1.0, -1.0)]


def draw_coef(rng, coefs):
    """One term coefficient: +-1 ("pm1") or a Gaussian integer from COMPLEX_COEFS ("complex")."""
    if coefs == "complex":
        return COMPLEX_COEFS[int(rng.integers(len(COMPLEX_COEFS)))]
    return (float(rng.choice([1.0, -1.0])), 0.0)


def config_c2(N=128, Lt=64, n_src=16, n_snk=16, n_loop4=384, n_loop2=16, n_corr=10, seed=1, coefs="pm1"):
    """c2: pi-pi I=2 correlator set.  4-meson loops TR_MM(MM1(src_a,snk_c), MM1(src_b,snk_d))
    with a<b, c!=d sampled without replacement; MM1 pairs shared across trees;
    plus 2-meson loops TR_MM(src_a, snk_c).  Each tree enters one or two of
    n_corr correlators with coefficient +-1 (coefs="complex": Gaussian integers)."""
    rng = np.random.default_rng(seed)
    b = Builder("c2_pipi_set_N%d_Lt%d" % (N, Lt), Lt, N, 1)
    src = [b.leaf(LEAF_M) for _ in range(n_src)]
    snk = [b.leaf(LEAF_M) for _ in range(n_snk)]
    combos = [(a, bb, c, d) for a in range(n_src) for bb in range(a + 1, n_src)
              for c in range(n_snk) for d in range(n_snk) if c != d]
    pick = rng.choice(len(combos), size=min(n_loop4, len(combos)), replace=False)
    # restrict MM1 pairs to a limited (src, snk) set so pairs are shared (F_v ~ 4-5)
    pair_pool = rng.permutation([(a, c) for a in range(n_src) for c in range(n_snk)])[:128]
    pool = [tuple(p) for p in pair_pool]
    trees = []
    for idx in range(len(pick)):
        (a, c) = pool[int(rng.integers(len(pool)))]
        (bb, d) = pool[int(rng.integers(len(pool)))]
        while (bb, d) == (a, c):
            (bb, d) = pool[int(rng.integers(len(pool)))]
        x = b.op(MM1, src[a], snk[c])
        y = b.op(MM1, src[bb], snk[d])
        trees.append(b.tree(b.op(TR_MM, x, y, share=False)))
    for i in range(n_loop2):
        a = i % n_src
        c = int(rng.integers(n_snk))
        trees.append(b.tree(b.op(TR_MM, src[a], snk[c], share=False)))
    for t in trees:
        cs = rng.choice(n_corr, size=int(rng.integers(1, 3)), replace=False)
        for c in sorted(int(x) for x in cs):
            b.term(c, t, *draw_coef(rng, coefs))
    _prune(b.w)
    return b.w


def config_traces(N=128, Lt=64, n_mes=128, n_traces=400, seed=1):
    """Diagnostic (not a BASELINE config): c2's trace stage alone — n_traces TR_MM of random
    distinct pairs of n_mes meson leaves (c2 traces 384 pairs of its 128 MM1 outputs)."""
    rng = np.random.default_rng(seed)
    b = Builder("traces_N%d_Lt%d_k%d" % (N, Lt, n_traces), Lt, N, 1)
    mes = [b.leaf(LEAF_M) for _ in range(n_mes)]
    seen = set()
    while len(seen) < n_traces:
        x, y = (int(v) for v in rng.choice(n_mes, size=2, replace=False))
        if (x, y) in seen:
            continue
        seen.add((x, y))
        b.term(len(seen) % 4, b.tree(b.op(TR_MM, mes[x], mes[y], share=False)))
    return b.w


def config_c3(N=64, Lt=32, S=64):
    """c3: single nucleon correlator: P = BM1(B_snk, tau1); X = BB2(P, B_src);
    root = TR_MM(X, tau2)."""
    b = Builder("c3_nucleon_N%d_Lt%d_S%d" % (N, Lt, S), Lt, N, S)
    bsnk = b.leaf(LEAF_B)
    bsrc = b.leaf(LEAF_B)
    tau1 = b.leaf(LEAF_M)
    tau2 = b.leaf(LEAF_M)
    p = b.op(BM1, bsnk, tau1)
    x = b.op(BB2, p, bsrc)
    t = b.tree(b.op(TR_MM, x, tau2, share=False))
    b.term(0, t)
    return b.w


def config_c4(N=128, Lt=1, S=64, n_snk=8, n_src=8, n_mes=16, n_trees=2000, p_dress=0.5,
              n_corr=8, seed=1):
    """c4: two-baryon system: root = TR_MM(BB2(Bsnk'_a, Bsrc_b), BB2(Bsnk'_c, Bsrc_d)),
    Bsnk' a sink leaf or (prob. p_dress) a shared dressing BM1(Bsnk, tau)."""
    rng = np.random.default_rng(seed)
    b = Builder("c4_two_baryon_N%d_Lt%d_S%d_k%d" % (N, Lt, S, n_trees), Lt, N, S)
    snk = [b.leaf(LEAF_B) for _ in range(n_snk)]
    src = [b.leaf(LEAF_B) for _ in range(n_src)]
    mes = [b.leaf(LEAF_M) for _ in range(n_mes)]
    dress_pool = [(a, m) for a in range(n_snk) for m in range(4)]

    def snk_prime():
        a = int(rng.integers(n_snk))
        if rng.random() < p_dress:
            (a, m) = dress_pool[int(rng.integers(len(dress_pool)))]
            return b.op(BM1, snk[a], mes[m])
        return snk[a]

    seen = set()
    trees = []
    tries = 0
    while len(trees) < n_trees and tries < 50 * n_trees:
        tries += 1
        x1, s1 = snk_prime(), int(rng.integers(n_src))
        x2, s2 = snk_prime(), int(rng.integers(n_src))
        key = (x1, s1, x2, s2)
        if key in seen or (x1, s1) == (x2, s2):
            continue
        seen.add(key)
        y1 = b.op(BB2, x1, src[s1])
        y2 = b.op(BB2, x2, src[s2])
        trees.append(b.tree(b.op(TR_MM, y1, y2, share=False)))
    for t in trees:
        b.term(int(rng.integers(n_corr)), t, float(rng.choice([1.0, -1.0])), 0.0)
    _prune(b.w)   # a dressing drawn for a rejected duplicate tree is unreferenced
    return b.w


def config_c5(N=256, Lt=128, n_mes=64, n_pairs=2000, n_trees=20000, zipf=1.1, n_corr=16, seed=1):
    """c5: meson-meson sweep: 4-meson loops TR_MM(MM1(p), MM1(q)) over n_pairs distinct
    MM1 pairs drawn with Zipf(zipf) popularity."""
    rng = np.random.default_rng(seed)
    b = Builder("c5_mxm_N%d_Lt%d_k%d" % (N, Lt, n_trees), Lt, N, 1)
    mes = [b.leaf(LEAF_M) for _ in range(n_mes)]
    pairs = set()
    while len(pairs) < n_pairs:
        x, y = (int(v) for v in rng.choice(n_mes, size=2, replace=False))
        pairs.add((x, y))
    pairs = sorted(pairs)
    rng.shuffle(pairs)
    w = 1.0 / np.arange(1, n_pairs + 1) ** zipf
    w /= w.sum()
    seen = set()
    trees = []
    tries = 0
    while len(trees) < n_trees and tries < 50 * n_trees:
        tries += 1
        i, j = (int(v) for v in rng.choice(n_pairs, size=2, p=w))
        if i == j or (i, j) in seen:
            continue
        seen.add((i, j))
        x = b.op(MM1, mes[pairs[i][0]], mes[pairs[i][1]])
        y = b.op(MM1, mes[pairs[j][0]], mes[pairs[j][1]])
        trees.append(b.tree(b.op(TR_MM, x, y, share=False)))
    for t in trees:
        b.term(int(rng.integers(n_corr)), t, float(rng.choice([1.0, -1.0])), 0.0)
    _prune(b.w)
    return b.w


def config_c6(N=32, Lt=8, S=64, n_snk=4, n_src=4, n_trees=200, p_meson=0.3, n_corr=4, seed=1, coefs="pm1"):
    """c6: tritium-like BxBxB system (Table II 'tritium': N = 32, O(N^5),
    8 leaves, every size class O(N^2) / O(N^3) / O(N^4)).  Each tree takes 3
    sink and 3 source baryon leaves and eliminates quark lines one contraction at a time
     through a tetraquark intermediate (reading T4-1..T4-4):
      X1 = BB1(snk_a, src_b)   [tetra]        Y1 = BT2(snk_c, X1)   [baryon]
      family A: X2 = BB1(Y1, src_d), Y2 = BT2(snk_e, X2), root = BB3(Y2, src_f)
      family B (prob. p_meson): M1 = BB2(Y1, src_d), M2 = BB2(snk_e, src_f), root = TR_MM(M1, M2)
    Identical contractions are shared across trees (prefixes X1, Y1 recur), duplicate trees are
    redrawn; each tree enters one correlator."""
    rng = np.random.default_rng(seed)
    b = Builder("c6_tritium_N%d_Lt%d_S%d_k%d" % (N, Lt, S, n_trees), Lt, N, S)
    snk = [b.leaf(LEAF_B) for _ in range(n_snk)]
    src = [b.leaf(LEAF_B) for _ in range(n_src)]
    seen = set()
    trees = []
    tries = 0
    while len(trees) < n_trees and tries < 50 * n_trees:
        tries += 1
        a, c, e = (int(rng.integers(n_snk)) for _ in range(3))
        bb, d, f = (int(rng.integers(n_src)) for _ in range(3))
        fam = 1 if rng.random() < p_meson else 0
        key = (fam, a, bb, c, d, e, f)
        if key in seen:
            continue
        seen.add(key)
        x1 = b.op(BB1, snk[a], src[bb])
        y1 = b.op(BT2, snk[c], x1)
        if fam == 0:
            x2 = b.op(BB1, y1, src[d])
            y2 = b.op(BT2, snk[e], x2)
            root = b.op(BB3, y2, src[f], share=False)
        else:
            m1 = b.op(BB2, y1, src[d])
            m2 = b.op(BB2, snk[e], src[f])
            root = b.op(TR_MM, m1, m2, share=False)
        trees.append(b.tree(root))
    for t in trees:
        b.term(int(rng.integers(n_corr)), t, *draw_coef(rng, coefs))
    _prune(b.w)
    return b.w
