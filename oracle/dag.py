"""O1 — contraction DAG formation (§II-B) and Eq. (1) ranks.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Plain Python; no code shared
with the product path.

Node fields follow P:162-183: child (ordered left/right), parents, type in
{LEAF, INTERIOR, ROOT} by degree, size.  A tree is the
closure of its root under operands (DESIGN reading T-5: trees are closed).
"""
from synth.dags import LEAF_M, LEAF_B, MM1, BM1, BB2, TR_MM, LEAF_X, OP_X, BB1, BT2, BB3, N_OPS, LEAF_OPS

LEAF, INTERIOR, ROOT = "LEAF", "INTERIOR", "ROOT"

MESON_KINDS = (LEAF_M, MM1, BB2)
BARYON_KINDS = (LEAF_B, BM1, BT2)
TETRA_KINDS = (BB1,)                     # reading T4-1: [Lt, N, N, N, N], no spin index
CONTRACT_ALL = (TR_MM, BB3)              # root-only kinds ("contract all")
GEMM_KINDS = (MM1, BM1, BB2, BB1, BT2)   # interior kinds ("exterior contract")


class OracleError(Exception):
    code = "INVAL"


class CycleError(OracleError):
    code = "CYCLE"


class InconsistentError(OracleError):
    code = "INCONSISTENT"


class MultiRootError(OracleError):
    code = "MULTIROOT"


class UnknownNodeError(OracleError):
    code = "UNKNOWN_NODE"


class Node:
    __slots__ = ("id", "op", "child", "parents", "size", "type", "rank")

    def __init__(self, nid, op, child, size):
        self.id = nid
        self.op = op
        self.child = child        # [] for leaves, [left, right] otherwise
        self.parents = []         # ascending id (reading S-3)
        self.size = size
        self.type = None
        self.rank = None


def tensor_size(op, Lt, N, S):
    """Bytes of the tensor a node of kind `op` holds (complex128 = 16 B):
    meson [Lt,N,N], baryon [Lt,S,N,N,N], tetra [Lt,N,N,N,N] (reading T4-1; the O(N^2) /
    O(N^3) / O(N^4) size classes of P:871-872), contract-all root [Lt] scalars (P:59 pins 16
    B/element)."""
    if op in MESON_KINDS:
        return 16 * Lt * N * N
    if op in BARYON_KINDS:
        return 16 * Lt * S * N ** 3
    if op in TETRA_KINDS:
        return 16 * Lt * N ** 4
    if op in CONTRACT_ALL:
        return 16 * Lt
    raise OracleError("abstract node needs an explicit size")


class Dag:
    """The contraction DAG G=(V,E) of P:159 plus the tree set and correlator terms."""

    def __init__(self, w):
        self.Lt, self.N, self.S = w.Lt, w.N, w.S
        self.nodes = {}
        for (nid, op, a, b, size) in w.nodes:
            if nid in self.nodes:
                raise InconsistentError("duplicate node id %d" % nid)
            if op not in range(N_OPS):
                raise OracleError("bad op %r" % (op,))
            abstract = op in (LEAF_X, OP_X)
            if abstract:
                if size <= 0:
                    raise OracleError("abstract node %d needs size > 0" % nid)
                sz = size
            else:
                sz = tensor_size(op, w.Lt, w.N, w.S)
                if size and size != sz:
                    raise InconsistentError("node %d size %d != shape size %d" % (nid, size, sz))
            if op in LEAF_OPS:
                if a != -1 or b != -1:
                    raise OracleError("leaf %d has operands" % nid)
                child = []
            else:
                if a == b:
                    raise OracleError("node %d: operands must differ" % nid)
                child = [a, b]
            self.nodes[nid] = Node(nid, op, child, sz)
        # edges (u, v): v depends on u
        for v in self.nodes.values():
            for u in v.child:
                if u not in self.nodes:
                    raise UnknownNodeError("node %d: unknown operand %d" % (v.id, u))
                self.nodes[u].parents.append(v.id)
        for u in self.nodes.values():
            u.parents.sort()
            if not u.child and not u.parents:
                raise InconsistentError("isolated node %d" % u.id)
            u.type = LEAF if not u.child else (ROOT if not u.parents else INTERIOR)
        self.ids = sorted(self.nodes)
        self.topo = self._toposort()
        self._check_shapes()
        self._ranks()
        # trees: members = closure of the root under operands
        self.trees = {}
        self.tree_ids = []
        root_owner = {}
        for (tid, r) in w.trees:
            if tid in self.trees:
                raise InconsistentError("duplicate tree id %d" % tid)
            if r not in self.nodes:
                raise UnknownNodeError("tree %d: unknown root %d" % (tid, r))
            if self.nodes[r].parents:
                raise InconsistentError("tree %d: root %d has parents" % (tid, r))
            if not self.nodes[r].child:
                raise InconsistentError("tree %d: root %d is a leaf" % (tid, r))
            if r in root_owner:
                raise MultiRootError("root %d shared by trees %d and %d" % (r, root_owner[r], tid))
            root_owner[r] = tid
            self.trees[tid] = (r, self._closure(r))
            self.tree_ids.append(tid)
        self.tree_ids.sort()
        for u in self.nodes.values():
            if u.type == ROOT and u.id not in root_owner:
                raise MultiRootError("parentless node %d is not the root of any tree" % u.id)
        self.ctree = {u: [] for u in self.nodes}
        for tid in self.tree_ids:
            for u in self.trees[tid][1]:
                self.ctree[u].append(tid)
        for u in self.nodes:
            if not self.ctree[u]:
                raise InconsistentError("node %d belongs to no tree" % u)
        self.terms = []
        for (c, t, re, im) in w.terms:
            if t not in self.trees:
                raise UnknownNodeError("term references unknown tree %d" % t)
            self.terms.append((c, t, complex(re, im)))

    # -- structure -----------------------------------------------------------------
    def _toposort(self):
        """Children before parents (iterative DFS); raises CycleError."""
        state = {}
        order = []
        for s in self.ids:
            if s in state:
                continue
            stack = [(s, 0)]
            state[s] = 1
            while stack:
                u, i = stack.pop()
                ch = self.nodes[u].child
                if i < len(ch):
                    stack.append((u, i + 1))
                    c = ch[i]
                    if state.get(c) == 1:
                        raise CycleError("cycle through %d" % c)
                    if c not in state:
                        state[c] = 1
                        stack.append((c, 0))
                else:
                    state[u] = 2
                    order.append(u)
        return order

    def _check_shapes(self):
        """Operand kinds per DESIGN readings V-1, T4-1..T4-3: MM1(M,M) BM1(B,M) BB2(B,B) TR_MM(M,M)
        BB1(B,B) BT2(B,T) BB3(B,B); the contract-all kinds (TR_MM, BB3) only as roots, the others
        never as roots."""
        for v in self.nodes.values():
            if v.op in LEAF_OPS:
                continue
            kinds = [self.nodes[c].op for c in v.child]
            if v.op == OP_X:
                ok = all(k in (LEAF_X, OP_X) for k in kinds)
            elif v.op in (MM1, TR_MM):
                ok = all(k in MESON_KINDS for k in kinds)
            elif v.op == BM1:
                ok = kinds[0] in BARYON_KINDS and kinds[1] in MESON_KINDS
            elif v.op in (BB2, BB1, BB3):
                ok = all(k in BARYON_KINDS for k in kinds)
            elif v.op == BT2:
                ok = kinds[0] in BARYON_KINDS and kinds[1] in TETRA_KINDS
            else:
                ok = False
            if not ok:
                raise InconsistentError("node %d: operand kinds %r do not fit op %d" % (v.id, kinds, v.op))
            if v.op in CONTRACT_ALL and v.parents:
                raise InconsistentError("contract-all node %d must be a root" % v.id)
            if v.op in GEMM_KINDS and not v.parents:
                raise InconsistentError("root %d must be a contract-all (TR_MM / BB3)" % v.id)

    def _ranks(self):
        """Eq. (1): rank(leaf)=0, else 1 + max child rank."""
        for u in self.topo:
            n = self.nodes[u]
            n.rank = 0 if not n.child else 1 + max(self.nodes[c].rank for c in n.child)

    def _closure(self, r):
        seen = set()
        stack = [r]
        while stack:
            u = stack.pop()
            if u in seen:
                continue
            seen.add(u)
            stack.extend(self.nodes[u].child)
        return frozenset(seen)

    # -- queries -------------------------------------------------------------------
    def contractions(self):
        return [u for u in self.ids if self.nodes[u].child]

    def n_edges(self):
        return sum(len(n.child) for n in self.nodes.values())

    def stats(self):
        """|V|, |E|, k, F_v, F_e exactly as defined at P:775-778."""
        V = len(self.nodes)
        E = self.n_edges()
        fv = sum(len(self.ctree[u]) for u in self.nodes) / V
        fe_num = 0
        for v in self.nodes.values():
            for u in v.child:
                fe_num += sum(1 for t in self.ctree[u] if v.id in self.trees[t][1])
        return {"V": V, "E": E, "k": len(self.trees), "n_contr": len(self.contractions()),
                "F_v": fv, "F_e": fe_num / E if E else 0.0,
                "max_rank": max(n.rank for n in self.nodes.values())}


def parse_text(text):
    """Parser of the text format in include/cc.h (oracle's own; errors carry line numbers)."""
    from synth.dags import Workload, OP_NAMES
    w = None
    names = {n: i for i, n in enumerate(OP_NAMES)}
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].split()
        if not line:
            continue
        try:
            if line[0] == "dims":
                w = Workload("parsed", int(line[1]), int(line[2]), int(line[3]))
            elif line[0] == "node":
                op = names[line[2]]
                rest = line[3:]
                a = b = -1
                if op not in LEAF_OPS:
                    a, b = int(rest[0]), int(rest[1])
                    rest = rest[2:]
                size = 0
                if rest:
                    if rest[0] != "size" or len(rest) != 2:
                        raise ValueError("trailing tokens")
                    size = int(rest[1])
                w.nodes.append((int(line[1]), op, a, b, size))
            elif line[0] == "tree":
                w.trees.append((int(line[1]), int(line[2])))
            elif line[0] == "term":
                w.terms.append((int(line[1]), int(line[2]), float(line[3]), float(line[4])))
            else:
                raise ValueError("unknown record %r" % line[0])
        except (ValueError, KeyError, IndexError, AttributeError) as e:
            raise OracleError("line %d: %s" % (ln, e))
    if w is None:
        raise OracleError("missing dims record")
    return w
