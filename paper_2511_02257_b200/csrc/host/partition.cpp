// Multi-GPU partition of a contraction DAG ("partitioning models ... for
// multi-GPU systems" is future work there; DESIGN.md §Multi-GPU gives this reading).
//
// TIME: every op is batched over time slices with no cross-t coupling (reading V-1), so
//   part p owns slices [p*Lt/n, (p+1)*Lt/n) of every tensor; nothing is replicated.
// TREES (reading M-1, round 2): the tree scheduler's selection order is a locality order
//   (trees sharing tensors are selected close together, §III-B); it is cut into n contiguous
//   chunks minimising the largest chunk's work — flops/8 of the distinct contractions in the
//   union of the chunk's tree closures (exact integers; abstract DAGs: 1 per contraction),
//   i.e. what the part executes, shared nodes replicated.  T* = the smallest bound for which
//   the first-fit cut needs at most n chunks (binary search; exact for min-max contiguous
//   partitions since a chunk's work only grows when it is extended); the parts are the
//   first-fit cut at T*, and while there are fewer than n chunks the one of largest work with
//   at least two trees (lowest index on ties) is split in half by tree count.
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
  const std::vector<int32_t>& sel = ts.tree_order;
  // contractions of every tree's closure, with their weights
  std::vector<std::vector<int32_t>> contr(g.trees.size());
  std::vector<int64_t> wt(g.nodes.size(), 0);
  for (size_t u = 0; u < g.nodes.size(); ++u)
    if (!g.nodes[u].leaf()) wt[u] = contraction_weight(g, g.nodes[u], g.Lt);
  for (int32_t t : sel)
    for (int32_t u : g.trees[size_t(t)].members)
      if (!g.nodes[size_t(u)].leaf()) contr[size_t(t)].push_back(u);
  std::vector<int32_t> stamp(g.nodes.size(), -1);
  int32_t next_stamp = 0;
  // work of a set of trees (distinct contractions of their closures)
  auto work_of = [&](const int32_t* t0, const int32_t* t1) {
    const int32_t s = next_stamp++;
    int64_t w = 0;
    for (const int32_t* t = t0; t != t1; ++t)
      for (int32_t u : contr[size_t(*t)])
        if (stamp[size_t(u)] != s) {
          stamp[size_t(u)] = s;
          w += wt[size_t(u)];
        }
    return w;
  };
  // first-fit cut at bound T: chunk start indices into sel; false if one tree exceeds T
  auto first_fit = [&](int64_t T, std::vector<size_t>& starts) {
    starts.clear();
    int32_t s = next_stamp++;
    int64_t w = 0;
    for (size_t i = 0; i < sel.size(); ++i) {
      const auto& mem = contr[size_t(sel[i])];
      int64_t add = 0;
      for (int32_t u : mem)
        if (stamp[size_t(u)] != s) add += wt[size_t(u)];
      if (!starts.empty() && w + add > T) {
        s = next_stamp++;
        w = 0;
        add = 0;
        for (int32_t u : mem) add += wt[size_t(u)];
        starts.push_back(i);
      } else if (starts.empty()) {
        starts.push_back(i);
      }
      if (add > T) return false;
      for (int32_t u : mem) stamp[size_t(u)] = s;
      w += add;
    }
    return true;
  };
  int64_t lo = 0;
  for (int32_t t : sel) lo = std::max(lo, work_of(&t, &t + 1));
  int64_t hi = sel.empty() ? 0 : work_of(sel.data(), sel.data() + sel.size());
  std::vector<size_t> starts;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (first_fit(mid, starts) && int64_t(starts.size()) <= n_parts) hi = mid;
    else lo = mid + 1;
  }
  if (!sel.empty()) first_fit(lo, starts);
  // chunks as [begin, end) index ranges; split the heaviest multi-tree chunk until n
  std::vector<std::pair<size_t, size_t>> chunks;
  for (size_t k = 0; k < starts.size(); ++k) chunks.push_back({starts[k], k + 1 < starts.size() ? starts[k + 1] : sel.size()});
  while (int64_t(chunks.size()) < n_parts) {
    int64_t best_w = -1;
    size_t best = chunks.size();
    for (size_t k = 0; k < chunks.size(); ++k) {
      if (chunks[k].second - chunks[k].first < 2) continue;
      const int64_t w = work_of(sel.data() + chunks[k].first, sel.data() + chunks[k].second);
      if (w > best_w) {
        best_w = w;
        best = k;
      }
    }
    if (best == chunks.size()) break;
    const size_t b = chunks[best].first, e = chunks[best].second, h = b + (e - b) / 2;
    chunks[best] = {b, h};
    chunks.insert(chunks.begin() + int64_t(best) + 1, {h, e});
  }
  std::vector<int32_t> part(g.trees.size(), 0);
  for (size_t k = 0; k < chunks.size(); ++k)
    for (size_t i = chunks[k].first; i < chunks[k].second; ++i) part[size_t(sel[i])] = int32_t(k);
  if (owner_tree) {
    std::vector<int32_t> owner(g.nodes.size(), -1);
    for (int32_t t : sel)
      for (int32_t u : g.trees[size_t(t)].members)
        if (owner[size_t(u)] < 0) owner[size_t(u)] = t;
    *owner_tree = std::move(owner);
  }
  if (sel_order) *sel_order = sel;
  return part;
}

}  // namespace cc
