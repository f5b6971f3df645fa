// Contraction DAG formation and validation (§II-B).
#include "dag.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>
#include <unordered_set>

namespace cc {

int64_t tensor_bytes(int op, int64_t Lt, int64_t N, int64_t S) {
  // complex128 = 16 B per element: meson [Lt,N,N], baryon [Lt,S,N,N,N], root [Lt]
  if (is_meson_kind(op)) return 16 * Lt * N * N;
  if (is_baryon_kind(op)) return 16 * Lt * S * N * N * N;
  if (is_tetra_kind(op)) return 16 * Lt * N * N * N * N;
  if (is_root_kind(op)) return 16 * Lt;
  throw Error(CC_E_INVAL, "abstract node needs an explicit size");
}

double node_flops(const Node& n, int64_t Lt, int64_t N, int64_t S) {
  // 8 real flops per complex multiply-add (4M real embedding, reading V-3)
  const double lt = double(Lt), nn = double(N), s = double(S);
  switch (n.op) {
    case CC_MM1: return 8.0 * lt * nn * nn * nn;
    case CC_BM1:
    case CC_BB2: return 8.0 * lt * s * nn * nn * nn * nn;
    case CC_TR_MM: return 8.0 * lt * nn * nn;
    case CC_BB1:
    case CC_BT2: return 8.0 * lt * s * nn * nn * nn * nn * nn;
    case CC_BB3: return 8.0 * lt * s * nn * nn * nn;
    default: return 0.0;
  }
}

double node_hbm_bytes(const Node& n, int64_t Lt, int64_t N, int64_t S) {
  const double lt = double(Lt), nn = double(N), s = double(S);
  switch (n.op) {
    case CC_MM1: return 48.0 * lt * nn * nn;
    case CC_BM1:
    case CC_BB2: return 16.0 * lt * (2.0 * s * nn * nn * nn + nn * nn);
    case CC_TR_MM: return 32.0 * lt * nn * nn;
    case CC_BB1: return 16.0 * lt * (2.0 * s * nn * nn * nn + nn * nn * nn * nn);     // 2 baryons in, tetra out
    case CC_BT2: return 16.0 * lt * (2.0 * s * nn * nn * nn + nn * nn * nn * nn);     // baryon + tetra in, baryon out
    case CC_BB3: return 32.0 * lt * s * nn * nn * nn;
    default: return 0.0;
  }
}

int32_t Dag::idx(int64_t id) const {
  auto it = index.find(id);
  if (it == index.end()) throw Error(CC_E_UNKNOWN_NODE, "unknown node id " + std::to_string(id));
  return it->second;
}

bool Dag::in_tree(int32_t u, int32_t t) const {
  const auto& v = ctree[u];
  return std::binary_search(v.begin(), v.end(), t);
}

static std::string S_(int64_t x) { return std::to_string(x); }

Dag::Dag(const Input& in, int32_t Lt_override, const std::vector<int64_t>* keep_trees) {
  Lt = Lt_override > 0 ? Lt_override : in.dims.Lt;
  N = in.dims.N;
  S = in.dims.S;
  if (in.dims.Lt <= 0 || N <= 0 || S <= 0) throw Error(CC_E_INVAL, "dims must be positive");

  // --- select the nodes (closure of the kept trees, or everything) -------------------
  std::unordered_map<int64_t, const cc_node*> byid;
  byid.reserve(in.nodes.size() * 2);
  for (const auto& n : in.nodes) {
    if (n.op < 0 || n.op >= CC_N_OPS) throw Error(CC_E_INVAL, "bad op for node " + S_(n.id));
    if (!byid.emplace(n.id, &n).second) throw Error(CC_E_INCONSISTENT, "duplicate node id " + S_(n.id));
  }
  std::vector<int64_t> ids;
  if (keep_trees) {
    std::unordered_set<int64_t> keep(keep_trees->begin(), keep_trees->end());
    std::unordered_set<int64_t> seen;
    std::vector<int64_t> stack;
    for (const auto& t : in.trees)
      if (keep.count(t.tree_id)) stack.push_back(t.root);
    while (!stack.empty()) {
      int64_t u = stack.back();
      stack.pop_back();
      if (!seen.insert(u).second) continue;
      auto it = byid.find(u);
      if (it == byid.end()) throw Error(CC_E_UNKNOWN_NODE, "unknown node id " + S_(u));
      if (!is_leaf_op(it->second->op)) {
        stack.push_back(it->second->a);
        stack.push_back(it->second->b);
      }
    }
    ids.assign(seen.begin(), seen.end());
  } else {
    for (const auto& n : in.nodes) ids.push_back(n.id);
  }
  std::sort(ids.begin(), ids.end());
  nodes.resize(ids.size());
  index.reserve(ids.size() * 2);
  for (size_t i = 0; i < ids.size(); ++i) index[ids[i]] = int32_t(i);

  bool any_abstract = false, any_typed = false;
  for (size_t i = 0; i < ids.size(); ++i) {
    const cc_node& src = *byid.at(ids[i]);
    Node& n = nodes[i];
    n.id = src.id;
    n.op = src.op;
    const bool abs_ = (src.op == CC_LEAF_X || src.op == CC_OP_X);
    (abs_ ? any_abstract : any_typed) = true;
    if (abs_) {
      if (src.size <= 0) throw Error(CC_E_INVAL, "abstract node " + S_(src.id) + " needs size > 0");
      n.size = src.size;
    } else {
      n.size = tensor_bytes(src.op, Lt, N, S);
      const int64_t full = tensor_bytes(src.op, in.dims.Lt, N, S);
      if (src.size && src.size != full)
        throw Error(CC_E_INCONSISTENT, "node " + S_(src.id) + " size does not match its shape");
    }
    if (is_leaf_op(src.op)) {
      if (src.a != -1 || src.b != -1) throw Error(CC_E_INVAL, "leaf " + S_(src.id) + " has operands");
    } else {
      if (src.a == src.b) throw Error(CC_E_INVAL, "node " + S_(src.id) + ": operands must differ");
      auto ia = index.find(src.a), ib = index.find(src.b);
      if (ia == index.end()) throw Error(CC_E_UNKNOWN_NODE, "node " + S_(src.id) + ": unknown operand " + S_(src.a));
      if (ib == index.end()) throw Error(CC_E_UNKNOWN_NODE, "node " + S_(src.id) + ": unknown operand " + S_(src.b));
      n.l = ia->second;
      n.r = ib->second;
    }
  }
  abstract = any_abstract;
  // parents in ascending id order (dense index order == id order)
  for (size_t v = 0; v < nodes.size(); ++v) {
    if (nodes[v].leaf()) continue;
    nodes[nodes[v].l].parents.push_back(int32_t(v));
    nodes[nodes[v].r].parents.push_back(int32_t(v));
    n_edges += 2;
  }
  for (auto& n : nodes) {
    std::sort(n.parents.begin(), n.parents.end());
    if (n.leaf() && n.parents.empty()) throw Error(CC_E_INCONSISTENT, "isolated node " + S_(n.id));
    n.type = n.leaf() ? LEAF : (n.parents.empty() ? ROOT : INTERIOR);
    if (!n.leaf()) ++n_contr;
  }

  // --- acyclicity + topological order (iterative DFS, children first) ---------------
  {
    std::vector<uint8_t> st(nodes.size(), 0);
    std::vector<std::pair<int32_t, int>> stack;
    topo.reserve(nodes.size());
    for (int32_t s = 0; s < int32_t(nodes.size()); ++s) {
      if (st[s]) continue;
      st[s] = 1;
      stack.push_back({s, 0});
      while (!stack.empty()) {
        auto& [u, i] = stack.back();
        const Node& n = nodes[u];
        const int nc = n.leaf() ? 0 : 2;
        if (i < nc) {
          int32_t c = (i == 0) ? n.l : n.r;
          ++i;
          if (st[c] == 1) throw Error(CC_E_CYCLE, "cycle through node " + S_(nodes[c].id));
          if (!st[c]) {
            st[c] = 1;
            stack.push_back({c, 0});
          }
        } else {
          st[u] = 2;
          topo.push_back(u);
          stack.pop_back();
        }
      }
    }
  }

  // --- operand kinds (reading V-1) ----------------------------------------------------
  if (any_abstract && any_typed) throw Error(CC_E_INCONSISTENT, "abstract and typed nodes mixed");
  for (const auto& n : nodes) {
    if (n.leaf()) continue;
    const int ka = nodes[n.l].op, kb = nodes[n.r].op;
    bool ok = false;
    switch (n.op) {
      case CC_OP_X: ok = true; break;
      case CC_MM1:
      case CC_TR_MM: ok = is_meson_kind(ka) && is_meson_kind(kb); break;
      case CC_BM1: ok = is_baryon_kind(ka) && is_meson_kind(kb); break;
      case CC_BB2:
      case CC_BB1:
      case CC_BB3: ok = is_baryon_kind(ka) && is_baryon_kind(kb); break;
      case CC_BT2: ok = is_baryon_kind(ka) && is_tetra_kind(kb); break;
      default: ok = false;
    }
    if (!ok) throw Error(CC_E_INCONSISTENT, "node " + S_(n.id) + ": operand kinds do not fit its op");
    if (is_root_kind(n.op) && !n.parents.empty())
      throw Error(CC_E_INCONSISTENT, "contract-all node " + S_(n.id) + " must be a root");
    if (is_gemm_kind(n.op) && n.parents.empty())
      throw Error(CC_E_INCONSISTENT, "root " + S_(n.id) + " must be a contract-all (TR_MM / BB3)");
  }

  // --- ranks, Eq. (1) ---------------------------------------------------------------------
  for (int32_t u : topo) {
    Node& n = nodes[u];
    n.rank = n.leaf() ? 0 : 1 + std::max(nodes[n.l].rank, nodes[n.r].rank);
    max_rank = std::max(max_rank, n.rank);
  }

  // --- trees: closure of the root under operands -------------------------------------
  std::vector<const cc_tree*> tin;
  {
    std::unordered_set<int64_t> keep;
    if (keep_trees) keep.insert(keep_trees->begin(), keep_trees->end());
    for (const auto& t : in.trees)
      if (!keep_trees || keep.count(t.tree_id)) tin.push_back(&t);
  }
  std::sort(tin.begin(), tin.end(), [](const cc_tree* a, const cc_tree* b) { return a->tree_id < b->tree_id; });
  tree_of_root.assign(nodes.size(), -1);
  std::vector<int32_t> mark(nodes.size(), -1);
  for (size_t ti = 0; ti < tin.size(); ++ti) {
    const cc_tree& t = *tin[ti];
    if (ti > 0 && tin[ti - 1]->tree_id == t.tree_id) throw Error(CC_E_INCONSISTENT, "duplicate tree id " + S_(t.tree_id));
    auto it = index.find(t.root);
    if (it == index.end()) throw Error(CC_E_UNKNOWN_NODE, "tree " + S_(t.tree_id) + ": unknown root " + S_(t.root));
    const int32_t r = it->second;
    if (!nodes[r].parents.empty()) throw Error(CC_E_INCONSISTENT, "tree " + S_(t.tree_id) + ": root has parents");
    if (nodes[r].leaf()) throw Error(CC_E_INCONSISTENT, "tree " + S_(t.tree_id) + ": root is a leaf");
    if (tree_of_root[r] >= 0) throw Error(CC_E_MULTIROOT, "root " + S_(t.root) + " shared by two trees");
    tree_of_root[r] = int32_t(trees.size());
    Tree tr{t.tree_id, r, {}};
    std::vector<int32_t> stack{r};
    const int32_t stamp = int32_t(trees.size());
    while (!stack.empty()) {
      int32_t u = stack.back();
      stack.pop_back();
      if (mark[u] == stamp) continue;
      mark[u] = stamp;
      tr.members.push_back(u);
      if (!nodes[u].leaf()) {
        stack.push_back(nodes[u].l);
        stack.push_back(nodes[u].r);
      }
    }
    std::sort(tr.members.begin(), tr.members.end());
    trees.push_back(std::move(tr));
  }
  for (const auto& n : nodes)
    if (n.type == ROOT && tree_of_root[index.at(n.id)] < 0)
      throw Error(CC_E_MULTIROOT, "parentless node " + S_(n.id) + " is not the root of any tree");
  ctree.assign(nodes.size(), {});
  for (int32_t t = 0; t < int32_t(trees.size()); ++t)
    for (int32_t u : trees[t].members) ctree[u].push_back(t);
  for (size_t u = 0; u < nodes.size(); ++u)
    if (ctree[u].empty()) throw Error(CC_E_INCONSISTENT, "node " + S_(nodes[u].id) + " belongs to no tree");

  // --- terms -------------------------------------------------------------------------------
  std::unordered_map<int64_t, int32_t> tix;
  for (int32_t t = 0; t < int32_t(trees.size()); ++t) tix[trees[t].tree_id] = t;
  for (const auto& x : in.terms) {
    auto it = tix.find(x.tree_id);
    if (it == tix.end()) {
      if (keep_trees) continue;  // term of a tree in another part
      throw Error(CC_E_UNKNOWN_NODE, "term references unknown tree " + S_(x.tree_id));
    }
    terms.push_back({x.corr_id, it->second, {x.re, x.im}});
    corr_ids.push_back(x.corr_id);
  }
  if (keep_trees) {
    // every correlator of the full input keeps its slot in each part (all-reduce layout)
    for (const auto& x : in.terms) corr_ids.push_back(x.corr_id);
  }
  std::sort(corr_ids.begin(), corr_ids.end());
  corr_ids.erase(std::unique(corr_ids.begin(), corr_ids.end()), corr_ids.end());
}

cc_dag_stats Dag::stats() const {
  cc_dag_stats s{};
  s.V = int64_t(nodes.size());
  s.E = n_edges;
  s.k = int64_t(trees.size());
  s.n_contr = n_contr;
  s.n_leaves = s.V - n_contr;
  s.max_rank = max_rank;
  s.n_corr = int64_t(corr_ids.size());
  // F_v, F_e exactly as defined at P:775-778
  double fv = 0;
  for (const auto& c : ctree) fv += double(c.size());
  s.F_v = s.V ? fv / double(s.V) : 0.0;
  double fe = 0;
  for (int32_t v = 0; v < int32_t(nodes.size()); ++v) {
    const Node& n = nodes[v];
    if (n.leaf()) continue;
    for (int32_t u : {n.l, n.r})
      for (int32_t t : ctree[u])
        if (in_tree(v, t)) fe += 1.0;
  }
  s.F_e = s.E ? fe / double(s.E) : 0.0;
  return s;
}

// --- text format (include/cc.h) ------------------------------------------------------------
Input parse_text_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw Error(CC_E_PARSE, "cannot open " + path);
  static const char* names[CC_N_OPS] = {"leafM", "leafB", "MM1", "BM1", "BB2", "TR_MM", "leafX", "OPX",
                                         "BB1", "BT2", "BB3"};
  Input in;
  bool have_dims = false;
  std::string line;
  int64_t ln = 0;
  while (std::getline(f, line)) {
    ++ln;
    auto h = line.find('#');
    if (h != std::string::npos) line.resize(h);
    std::istringstream ss(line);
    std::vector<std::string> tok;
    for (std::string t; ss >> t;) tok.push_back(t);
    if (tok.empty()) continue;
    auto fail = [&](const std::string& m) { throw Error(CC_E_PARSE, "line " + S_(ln) + ": " + m); };
    auto num = [&](size_t i) -> int64_t {
      if (i >= tok.size()) fail("missing field");
      try { size_t p; int64_t v = std::stoll(tok[i], &p); if (p != tok[i].size()) fail("bad integer " + tok[i]); return v; }
      catch (const std::logic_error&) { fail("bad integer " + tok[i]); }
      return 0;
    };
    auto real = [&](size_t i) -> double {
      if (i >= tok.size()) fail("missing field");
      try { size_t p; double v = std::stod(tok[i], &p); if (p != tok[i].size()) fail("bad number " + tok[i]); return v; }
      catch (const std::logic_error&) { fail("bad number " + tok[i]); }
      return 0;
    };
    if (tok[0] == "dims") {
      in.dims = {int32_t(num(1)), int32_t(num(2)), int32_t(num(3))};
      have_dims = true;
    } else if (tok[0] == "node") {
      if (tok.size() < 3) fail("missing field");
      int op = -1;
      for (int i = 0; i < CC_N_OPS; ++i)
        if (tok[2] == names[i]) op = i;
      if (op < 0) fail("unknown op " + tok[2]);
      cc_node n{num(1), op, 0, -1, -1, 0};
      size_t p = 3;
      if (!is_leaf_op(op)) { n.a = num(3); n.b = num(4); p = 5; }
      if (p < tok.size()) {
        if (tok[p] != "size" || p + 2 != tok.size()) fail("trailing tokens");
        n.size = num(p + 1);
      }
      in.nodes.push_back(n);
    } else if (tok[0] == "tree") {
      in.trees.push_back({num(1), num(2)});
    } else if (tok[0] == "term") {
      in.terms.push_back({num(1), num(2), real(3), real(4)});
    } else {
      fail("unknown record " + tok[0]);
    }
  }
  if (!have_dims) throw Error(CC_E_PARSE, "missing dims record");
  return in;
}

}  // namespace cc
