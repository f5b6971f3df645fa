// The paper's two schedulers (§III).  Both return the contraction order as
// dense node indices; leaf loads are lazy (reading G-6) and happen in the plan.
#pragma once
#include <vector>

#include "dag.hpp"

namespace cc {

// Alg. 1-3, sibling scheduler (§III-A); O(V+E).
std::vector<int32_t> sibling_schedule(const Dag& g);

struct TreeSchedule {
  std::vector<int32_t> order;       // contractions
  std::vector<int32_t> tree_order;  // selected tree indices, in selection order
};
// Alg. 4-8, tree scheduler (§III-B); O(kE).
TreeSchedule tree_schedule(const Dag& g);

// RS-GS-like baseline (Redstar's similarity sort, §II-A; readings R-1..R-4):
// the similarity chain of tree indices and the resulting contraction order.
std::vector<int32_t> rsgs_tree_chain(const Dag& g);
std::vector<int32_t> rsgs_schedule(const Dag& g);

}  // namespace cc
