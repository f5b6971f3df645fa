// Tree scheduler, Alg. 4-8 (§III-B).
//
// Gains: tgain(T) = cgain(T) + sum of igain(T,u) over T's unprocessed members;
// the scheduler repeatedly takes the alive tree of maximum tgain (ties: lowest tree id,
// reading T-1), processes its AVAIL members in post-order from the root, left operand
// first (T-2), and updates the gains of the other trees incrementally through tau/delta
// (PROCESS-CHILD cases 1.a / 2.a; PROCESS-NODE coarse gains).
// Corrections of the printed pseudocode: G-2 (Alg. 5 adds igain), G-3 (Alg. 7 updates
// x.outAv), G-4 (INMEM).  The max is kept in a tournament tree refreshed lazily before
// each selection, so a run is O(kE + k log k).
#include <algorithm>
#include <climits>

#include "sched.hpp"

namespace cc {
namespace {

enum St : uint8_t { AVAIL, INMEM, RELEASED };

struct Entry {            // tau(u,T), delta(u,T) for one successor tree T of u
  int32_t tree;
  int32_t tau, delta;
  bool in_pred;           // u in T.pred  (tau > 0)
};

struct TreeSched {
  const Dag& g;
  const int32_t k;
  std::vector<uint8_t> st;
  std::vector<int32_t> out_av;                  // |u.outAv|
  std::vector<int64_t> igain_flat;              // aligned with g.ctree[u]
  std::vector<size_t> igain_off;
  std::vector<std::vector<Entry>> succ;         // per node: its tau/delta entries
  std::vector<int64_t> tgain, cgain;
  std::vector<uint8_t> alive, dirty;
  std::vector<int32_t> dirty_list;
  // tournament tree over trees: best tree index of each subtree
  int32_t leaves = 1;
  std::vector<int32_t> seg;
  std::vector<int32_t> stamp;                   // scratch for PROCESS-NODE's set S
  int32_t stamp_id = 0;
  std::vector<int32_t> pos_in_s;
  TreeSchedule out;

  explicit TreeSched(const Dag& g_) : g(g_), k(int32_t(g_.trees.size())) {}

  bool better(int32_t a, int32_t b) const {     // is tree a preferred over tree b
    if (a < 0) return false;
    if (b < 0) return true;
    const bool la = alive[a], lb = alive[b];
    if (la != lb) return la;
    if (tgain[a] != tgain[b]) return tgain[a] > tgain[b];
    return a < b;                                // T-1
  }
  void seg_update(int32_t t) {
    int32_t i = t + leaves;
    seg[i] = t;
    for (i >>= 1; i >= 1; i >>= 1) seg[i] = better(seg[2 * i], seg[2 * i + 1]) ? seg[2 * i] : seg[2 * i + 1];
  }
  void touch(int32_t t) {
    if (!dirty[t]) {
      dirty[t] = 1;
      dirty_list.push_back(t);
    }
  }

  // Alg. 5 TR-INIT
  void init() {
    const size_t n = g.nodes.size();
    st.assign(n, AVAIL);
    out_av.resize(n);
    igain_off.resize(n + 1);
    succ.assign(n, {});
    tgain.assign(size_t(k), 0);
    cgain.assign(size_t(k), 0);
    alive.assign(size_t(k), 1);
    dirty.assign(size_t(k), 0);
    size_t total = 0;
    for (size_t u = 0; u < n; ++u) {
      out_av[u] = int32_t(g.nodes[u].parents.size());   // u.outAv = u.parents
      igain_off[u] = total;
      total += g.ctree[u].size();
    }
    igain_off[n] = total;
    igain_flat.resize(total);
    for (size_t u = 0; u < n; ++u) {
      const auto& ct = g.ctree[u];
      for (size_t i = 0; i < ct.size(); ++i) {
        const int32_t t = ct[i];
        // g(u,T) = |outAv(u)| - #{(u,v) in E : T in v.ctree}
        int32_t gv = out_av[u];
        for (int32_t v : g.nodes[u].parents)
          if (g.in_tree(v, t)) --gv;
        const int64_t ig = (gv == 0) ? 0 : -g.nodes[u].size;
        igain_flat[igain_off[u] + i] = ig;
        tgain[size_t(t)] += ig;                           // G-2
      }
    }
    while (leaves < std::max(k, 1)) leaves <<= 1;
    seg.assign(size_t(2 * leaves), -1);
    for (int32_t t = 0; t < k; ++t) seg[size_t(t + leaves)] = t;
    for (int32_t i = leaves - 1; i >= 1; --i)
      seg[size_t(i)] = better(seg[size_t(2 * i)], seg[size_t(2 * i + 1)]) ? seg[size_t(2 * i)] : seg[size_t(2 * i + 1)];
    stamp.assign(size_t(k), -1);
    pos_in_s.assign(size_t(k), -1);
  }

  // Alg. 7 PROCESS-CHILD(u, x)
  void process_child(int32_t u, int32_t x) {
    const int64_t size = g.nodes[x].size;
    const auto& cu = g.ctree[u];
    size_t j = 0;
    for (Entry& e : succ[x]) {                    // entries sorted by tree index
      if (!e.in_pred) continue;                   // T_i : x in T_i.pred
      const int32_t t = e.tree;
      while (j < cu.size() && cu[j] < t) ++j;
      const bool u_in_t = (j < cu.size() && cu[j] == t);
      if (u_in_t) {
        if (e.tau == 1 && e.delta == 0) {         // case 1.a
          cgain[t] -= size;
          tgain[t] -= size;
          touch(t);
        }
        if (--e.tau < 0) throw Error(CC_E_STATE, "tree scheduler: tau underflow");
        if (e.tau == 0) e.in_pred = false;        // T_i.pred -= x
      } else {
        if (e.delta == 1) {                       // case 2.a
          cgain[t] += size;
          tgain[t] += size;
          touch(t);
        }
        if (--e.delta < 0) throw Error(CC_E_STATE, "tree scheduler: delta underflow");
      }
    }
    if (--out_av[x] == 0) st[x] = RELEASED;       // x.outAv = x.outAv - u   (G-3)
  }

  // Alg. 8 PROCESS-NODE(u)
  void process_node(int32_t u) {
    const Node& n = g.nodes[u];
    const auto& cu = g.ctree[u];
    for (size_t i = 0; i < cu.size(); ++i) {     // l.1-2
      tgain[cu[i]] -= igain_flat[igain_off[u] + i];
      touch(cu[i]);
    }
    ++stamp_id;                                   // l.3-12: set S over trees of u.outAv
    std::vector<Entry>& es = succ[u];
    const int32_t n_out = out_av[u];
    for (int32_t v : n.parents) {
      if (st[v] != AVAIL) throw Error(CC_E_STATE, "tree scheduler: processed parent of an AVAIL node");
      for (int32_t t : g.ctree[v]) {
        if (stamp[t] != stamp_id) {
          stamp[t] = stamp_id;
          pos_in_s[t] = int32_t(es.size());
          es.push_back({t, 0, n_out, true});      // tau = 0, delta = |outAv|, pred += u
        }
        Entry& e = es[size_t(pos_in_s[t])];
        --e.delta;
        ++e.tau;
      }
    }
    for (Entry& e : es) {                         // l.13-16 coarse gains
      if (e.delta == 0) {
        cgain[e.tree] += n.size;
        tgain[e.tree] += n.size;
        touch(e.tree);
      }
    }
    std::sort(es.begin(), es.end(), [](const Entry& a, const Entry& b) { return a.tree < b.tree; });
    st[u] = (out_av[u] == 0) ? RELEASED : INMEM;  // l.17-20 (G-4)
  }

  // Alg. 6 PROCESS-CTREE(T): post-order from the root, left first, AVAIL members (T-2)
  void process_ctree(int32_t t) {
    std::vector<std::pair<int32_t, int>> stack{{g.trees[t].root, 0}};
    std::vector<int32_t> post;
    ++stamp_id;
    // visited marks for this tree walk live in a per-node vector reused across trees
    while (!stack.empty()) {
      auto& [u, i] = stack.back();
      if (i == 0) {
        if (visit_mark[u] == stamp_id || st[u] != AVAIL) {
          stack.pop_back();
          continue;
        }
        visit_mark[u] = stamp_id;
      }
      const Node& n = g.nodes[u];
      if (!n.leaf() && i < 2) {
        const int32_t c = (i == 0) ? n.l : n.r;
        ++i;
        stack.push_back({c, 0});
      } else {
        post.push_back(u);
        stack.pop_back();
      }
    }
    for (int32_t u : post) {
      const Node& n = g.nodes[u];
      if (!n.leaf()) {
        process_child(u, n.l);
        process_child(u, n.r);
        out.order.push_back(u);
      }
      process_node(u);
    }
  }
  std::vector<int32_t> visit_mark;

  TreeSchedule run() {
    init();
    visit_mark.assign(g.nodes.size(), -1);
    out.order.reserve(size_t(g.n_contr));
    out.tree_order.reserve(size_t(k));
    for (int32_t it = 0; it < k; ++it) {          // Alg. 4
      for (int32_t t : dirty_list) {
        dirty[t] = 0;
        seg_update(t);
      }
      dirty_list.clear();
      const int32_t t = seg[1];
      if (t < 0 || !alive[t]) throw Error(CC_E_STATE, "tree scheduler: no alive tree");
      out.tree_order.push_back(t);
      process_ctree(t);
      alive[t] = 0;                               // A = A - T'
      touch(t);
    }
    return std::move(out);
  }
};

}  // namespace

TreeSchedule tree_schedule(const Dag& g) { return TreeSched(g).run(); }

}  // namespace cc
