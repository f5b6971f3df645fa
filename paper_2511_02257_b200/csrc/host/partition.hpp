// Multi-GPU partitions.
#pragma once
#include <vector>

#include "dag.hpp"

namespace cc {
// Part index of every tree (indexed like g.trees) for a TREES split into n_parts;
// sel_order (optional) receives the tree-scheduler selection order used, owner_tree (optional)
// the first selected tree containing each node (-1: in no tree).
std::vector<int32_t> tree_parts(const Dag& g, int32_t n_parts, std::vector<int32_t>* sel_order,
                                std::vector<int32_t>* owner_tree = nullptr);
// flops / 8 of one contraction at lt time slices (abstract DAGs: 1)
int64_t contraction_weight(const Dag& g, const Node& n, int64_t lt);
}  // namespace cc
