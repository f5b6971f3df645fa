// RS-GS-like baseline scheduler: Redstar's similarity sort of contraction
// trees (§II-A; the RS-GS baseline of §IV) under readings
// R-1..R-4:
//   R-1 similarity = Jaccard |A∩B| / |A∪B| of the trees' member sets (closures, leaves in);
//   R-2 greedy chain from the lowest tree id, next = unvisited tree most similar to the last
//       one, ties -> lowest id, fractions compared exactly by cross-multiplication;
//   R-3 each tree contributes its uncontracted non-leaf members in T-2 order (post-order from
//       the root, left operand first, not descending into contracted nodes);
//   R-4 Redstar's edge-frequency/complexity path selection has nothing to choose: contraction
//       paths are fixed by the input DAG.
// Cost: O(sum over chain steps of (members of the last tree x trees per member)) with an
// inverted index, plus an ordered set of unvisited ids for all-zero steps.
#include <set>
#include <vector>

#include "sched.hpp"

namespace cc {

std::vector<int32_t> rsgs_tree_chain(const Dag& g) {
  const int32_t k = int32_t(g.trees.size());
  std::vector<int32_t> chain;
  if (k == 0) return chain;
  std::set<int32_t> unvisited;
  for (int32_t t = 0; t < k; ++t) unvisited.insert(t);
  std::vector<int64_t> inter(size_t(k), 0);
  std::vector<uint8_t> visited(size_t(k), 0);
  std::vector<int32_t> touched;
  int32_t cur = 0;   // trees are sorted by id: index 0 is the lowest id
  for (;;) {
    chain.push_back(cur);
    visited[size_t(cur)] = 1;
    unvisited.erase(cur);
    if (unvisited.empty()) break;
    touched.clear();
    for (int32_t u : g.trees[size_t(cur)].members)
      for (int32_t t : g.ctree[size_t(u)])
        if (!visited[size_t(t)]) {
          if (inter[size_t(t)] == 0) touched.push_back(t);
          ++inter[size_t(t)];
        }
    if (touched.empty()) {
      cur = *unvisited.begin();   // every similarity is 0: lowest unvisited id
      continue;
    }
    const int64_t mc = int64_t(g.trees[size_t(cur)].members.size());
    int32_t best = -1;
    int64_t ba = 0, bb = 1;
    for (int32_t t : touched) {
      const int64_t a = inter[size_t(t)];
      const int64_t b = mc + int64_t(g.trees[size_t(t)].members.size()) - a;
      // a/b > ba/bb, or equal with a lower index (tree index order == id order)
      if (best < 0 || a * bb > ba * b || (a * bb == ba * b && t < best)) {
        best = t;
        ba = a;
        bb = b;
      }
    }
    for (int32_t t : touched) inter[size_t(t)] = 0;
    cur = best;
  }
  return chain;
}

std::vector<int32_t> rsgs_schedule(const Dag& g) {
  std::vector<int32_t> order;
  order.reserve(size_t(g.n_contr));
  std::vector<uint8_t> done(g.nodes.size(), 0), seen(g.nodes.size(), 0);
  std::vector<int32_t> seen_list;
  for (int32_t t : rsgs_tree_chain(g)) {
    // R-3 / T-2: post-order from the root, left operand first
    std::vector<std::pair<int32_t, int>> stack{{g.trees[size_t(t)].root, 0}};
    seen_list.clear();
    while (!stack.empty()) {
      auto& [u, i] = stack.back();
      const Node& n = g.nodes[size_t(u)];
      if (i == 0) {
        if (seen[size_t(u)] || done[size_t(u)]) {
          stack.pop_back();
          continue;
        }
        seen[size_t(u)] = 1;
        seen_list.push_back(u);
      }
      const int32_t c = i == 0 ? n.l : (i == 1 ? n.r : -1);
      if (c >= 0) {
        ++i;
        stack.push_back({c, 0});
      } else {
        if (!n.leaf()) {
          done[size_t(u)] = 1;
          order.push_back(u);
        }
        stack.pop_back();
      }
    }
    for (int32_t u : seen_list) seen[size_t(u)] = 0;
  }
  return order;
}

}  // namespace cc
