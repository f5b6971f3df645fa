// Multi-GPU partition of a contraction DAG ("partitioning models ... for
// multi-GPU systems" is future work there; DESIGN.md §Multi-GPU gives this reading).
//
// TIME: every op is batched over time slices with no cross-t coupling (reading V-1), so
//   part p owns slices [p*Lt/n, (p+1)*Lt/n) of every tensor; nothing is replicated.
// TREES: the tree scheduler's selection order is a locality order (trees sharing tensors
//   are selected close together, §III-B).  Each tree is weighted by the flops of the
//   contractions first executed while processing it (flops/8, exact integers; abstract
//   DAGs: number of contractions), and tree i (prefix weight P_i, weight w_i, total W)
//   goes to part min(n-1, floor(n * (2 P_i + w_i) / (2 W))) — contiguous, flop-balanced
//   chunks.  Each part keeps the closure of its trees, so shared nodes are replicated.
// GRID (reading M-2): TREES part p / n_time restricted to TIME part p % n_time.
// Owners (readings M-3, E-11): the owner part of a node is the part of the first selected
//   tree containing it; replicated work / leaf bytes of a part are those it holds but does
//   not own, and a leaf's owner is the rank that loads it over PCIe for the others.
#include <algorithm>

#include "partition.hpp"
#include "sched.hpp"

namespace cc {

int64_t contraction_weight(const Dag& g, const Node& n, int64_t lt) {
  if (g.abstract) return 1;
  const int64_t nn = g.N, s = g.S;
  switch (n.op) {
    case CC_MM1: return lt * nn * nn * nn;
    case CC_BM1:
    case CC_BB2: return lt * s * nn * nn * nn * nn;
    case CC_TR_MM: return lt * nn * nn;
    case CC_BB1:
    case CC_BT2: return lt * s * nn * nn * nn * nn * nn;
    case CC_BB3: return lt * s * nn * nn * nn;
    default: return 1;
  }
}

std::vector<int32_t> tree_parts(const Dag& g, int32_t n_parts, std::vector<int32_t>* sel_order,
                                std::vector<int32_t>* owner_tree) {
  TreeSchedule ts = tree_schedule(g);
  // first-execution weight of each selected tree
  std::vector<int64_t> w(g.trees.size(), 0);
  // a contraction is executed while processing the first selected tree containing it
  std::vector<int32_t> owner(g.nodes.size(), -1);
  for (int32_t t : ts.tree_order)
    for (int32_t u : g.trees[t].members)
      if (owner[u] < 0) owner[u] = t;
  for (int32_t u : ts.order) w[size_t(owner[u])] += contraction_weight(g, g.nodes[u], g.Lt);
  __int128 W = 0;
  for (int32_t t : ts.tree_order) W += w[size_t(t)];
  std::vector<int32_t> part(g.trees.size(), 0);
  __int128 P = 0;
  for (int32_t t : ts.tree_order) {
    int64_t p = 0;
    if (W > 0) {
      const __int128 num = __int128(n_parts) * (2 * P + w[size_t(t)]);
      p = int64_t(num / (2 * W));
    }
    part[size_t(t)] = int32_t(std::min<int64_t>(n_parts - 1, p));
    P += w[size_t(t)];
  }
  if (sel_order) *sel_order = ts.tree_order;
  if (owner_tree) *owner_tree = std::move(owner);
  return part;
}

}  // namespace cc
