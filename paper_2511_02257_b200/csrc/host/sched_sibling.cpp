// Sibling scheduler, Alg. 1-3 (§III-A).
//
// Rank-priority queues Q_1..Q_q; the highest non-empty queue is served;
// when all are empty a WAITING leaf is picked (reading S-1: the lowest-id one).  Node
// processing (Alg. 2) releases children at rs == 0 and, for each parent (ascending id,
// S-3), either prop-downs the sibling subtree (rp == 1, Alg. 3, left then right, S-4)
// or enqueues the parent (rp == 0).  FIFO within a queue (S-2).  Every node is
// processed once, so the run is O(V + E).
#include <deque>

#include "sched.hpp"

namespace cc {
namespace {

enum St : uint8_t { WAITING, QUEUED, INMEM, RELEASED };

struct Sibling {
  const Dag& g;
  std::vector<int32_t> rs, rp;
  std::vector<uint8_t> st;
  std::vector<std::deque<int32_t>> q;   // q[r] = Q_r, r in 1..max_rank
  std::vector<int32_t> order;

  explicit Sibling(const Dag& g_) : g(g_) {
    const size_t n = g.nodes.size();
    rs.resize(n);
    rp.resize(n);
    st.assign(n, WAITING);
    for (size_t u = 0; u < n; ++u) {
      rs[u] = int32_t(g.nodes[u].parents.size());     // rs = |u.parents|
      rp[u] = g.nodes[u].leaf() ? 0 : 2;               // rp = |u.child|
    }
    q.resize(size_t(g.max_rank) + 1);
  }

  // Alg. 3 SB-PROP-DOWN
  void prop_down(int32_t u) {
    // iterative form of the recursion "prop_down(left); prop_down(right)" that keeps
    // its visiting order: a node's left subtree completes before its right one starts
    std::vector<int32_t> stack{u};
    while (!stack.empty()) {
      int32_t x = stack.back();
      stack.pop_back();
      if (st[x] != WAITING) continue;                    // l.1-3
      const Node& n = g.nodes[x];
      if (n.leaf()) {                                    // l.4-7
        process(x);
        continue;
      }
      stack.push_back(n.r);                              // l.9 right runs after l.8 left
      stack.push_back(n.l);
    }
  }

  // Alg. 2 SB-PROCESS
  void process(int32_t u) {
    const Node& n = g.nodes[u];
    if (!n.leaf()) order.push_back(u);                   // l.1-4 contract / bring to memory
    st[u] = INMEM;                                       // l.5
    if (!n.leaf()) {                                     // l.6-12
      for (int32_t v : {n.l, n.r})
        if (--rs[v] == 0) st[v] = RELEASED;
      if (n.type == ROOT) st[u] = RELEASED;
    }
    for (int32_t v : n.parents) {                        // l.13-21, ascending id
      --rp[v];
      if (rp[v] == 1) {
        const Node& p = g.nodes[v];
        const int32_t w = (p.l == u) ? p.r : p.l;        // sibling of u under v
        if (st[w] == WAITING) prop_down(w);
      } else if (rp[v] == 0) {
        q[size_t(g.nodes[v].rank)].push_back(v);         // ENQUEUE(Q_{v.rank}, v)
        st[v] = QUEUED;
      }
    }
  }

  std::vector<int32_t> run() {
    int32_t leaf_cursor = 0;
    const int32_t n = int32_t(g.nodes.size());
    order.reserve(size_t(g.n_contr));
    while (int64_t(order.size()) < g.n_contr) {          // Alg. 1
      int r = g.max_rank;
      while (r >= 1 && q[size_t(r)].empty()) --r;
      int32_t u;
      if (r < 1) {
        while (leaf_cursor < n && !(g.nodes[leaf_cursor].leaf() && st[leaf_cursor] == WAITING)) ++leaf_cursor;
        if (leaf_cursor == n) throw Error(CC_E_STATE, "sibling scheduler stuck: no WAITING leaf");
        u = leaf_cursor;
      } else {
        u = q[size_t(r)].front();
        q[size_t(r)].pop_front();
      }
      process(u);
    }
    return std::move(order);
  }
};

}  // namespace

std::vector<int32_t> sibling_schedule(const Dag& g) { return Sibling(g).run(); }

}  // namespace cc
