// Contraction DAG G=(V,E) (§II-B) with ranks (Eq. 1)
// and tree memberships (u.ctree).  Host-side, single-threaded.
#pragma once
#include <cstdint>
#include <complex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "cc.h"

namespace cc {

struct Error : std::runtime_error {
  cc_status status;
  Error(cc_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

enum NodeType : uint8_t { LEAF = 0, INTERIOR = 1, ROOT = 2 };

inline bool is_leaf_op(int op) { return op == CC_LEAF_M || op == CC_LEAF_B || op == CC_LEAF_X; }
inline bool is_meson_kind(int op) { return op == CC_LEAF_M || op == CC_MM1 || op == CC_BB2; }
inline bool is_baryon_kind(int op) { return op == CC_LEAF_B || op == CC_BM1 || op == CC_BT2; }
inline bool is_tetra_kind(int op) { return op == CC_BB1; }
inline bool is_root_kind(int op) { return op == CC_TR_MM || op == CC_BB3; }   // "contract all"
inline bool is_gemm_kind(int op) {
  return op == CC_MM1 || op == CC_BM1 || op == CC_BB2 || op == CC_BB1 || op == CC_BT2;
}

struct Node {
  int64_t id = 0;
  int32_t op = 0;
  int32_t l = -1, r = -1;          // dense operand indices (left, right), -1 for leaves
  std::vector<int32_t> parents;    // dense indices, ascending id (reading S-3)
  int64_t size = 0;                // bytes (or explicit abstract units)
  int32_t rank = 0;                // Eq. (1)
  NodeType type = LEAF;
  bool leaf() const { return l < 0; }
};

struct Tree {
  int64_t tree_id;
  int32_t root;                    // dense node index
  std::vector<int32_t> members;    // closure of the root under operands, ascending
};

struct Term { int64_t corr_id; int32_t tree; std::complex<double> coef; };

// The raw input as given to cc_load_dag (kept so partitions can rebuild the DAG).
struct Input {
  cc_dims dims{0, 0, 0};
  std::vector<cc_node> nodes;
  std::vector<cc_tree> trees;
  std::vector<cc_term> terms;
};

class Dag {
 public:
  // Builds and validates.  Lt_override > 0 replaces dims.Lt for the tensor sizes (TIME part).
  // keep_trees (optional): only these tree ids (and their closures / terms) are kept.
  Dag(const Input& in, int32_t Lt_override = 0, const std::vector<int64_t>* keep_trees = nullptr);

  int32_t Lt, N, S;
  std::vector<Node> nodes;                       // sorted by id
  std::unordered_map<int64_t, int32_t> index;    // id -> dense index
  std::vector<int32_t> topo;                     // children before parents
  std::vector<Tree> trees;                       // sorted by tree id
  std::vector<std::vector<int32_t>> ctree;       // per node: tree indices, ascending
  std::vector<Term> terms;                       // input order
  std::vector<int64_t> corr_ids;                 // distinct correlator ids, ascending
  std::vector<int32_t> tree_of_root;             // per node: tree index if root else -1
  bool abstract = false;                         // contains LEAF_X / OP_X
  int32_t max_rank = 0;
  int64_t n_contr = 0, n_edges = 0;

  int32_t idx(int64_t id) const;
  bool in_tree(int32_t u, int32_t t) const;      // t in ctree[u] (binary search)
  cc_dag_stats stats() const;
};

int64_t tensor_bytes(int op, int64_t Lt, int64_t N, int64_t S);
double node_flops(const Node& n, int64_t Lt, int64_t N, int64_t S);
double node_hbm_bytes(const Node& n, int64_t Lt, int64_t N, int64_t S);

Input parse_text_file(const std::string& path);

}  // namespace cc
