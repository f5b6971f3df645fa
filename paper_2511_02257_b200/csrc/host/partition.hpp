// Multi-GPU partitions.
#pragma once
#include <vector>

#include "dag.hpp"

namespace cc {
// Part index of every tree (indexed like g.trees) for a TREES split into n_parts;
// sel_order (optional) receives the tree-scheduler selection order used.
std::vector<int32_t> tree_parts(const Dag& g, int32_t n_parts, std::vector<int32_t>* sel_order);
}  // namespace cc
