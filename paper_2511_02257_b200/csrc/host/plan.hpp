// Memory model (§II-C), LRU device plan (MemHC-style eviction) and physical placement.
#pragma once
#include <map>
#include <set>
#include <vector>

#include "dag.hpp"

namespace cc {

// §II-C: M_0..M_n after releases; transient_i after producing c_i's output
// (reading G-5); leaves loaded lazily (G-6).
struct ModelTrace {
  std::vector<int64_t> M, transient;
  int64_t peak = 0, transient_peak = 0;
};
ModelTrace simulate_model(const Dag& g, const std::vector<int32_t>& order);
// Throws CC_E_INVAL when `order` is not a valid schedule of g.
void check_order(const Dag& g, const std::vector<int32_t>& order);

// OP_P2P_OUT: eviction copied to the peer-HBM tier; OP_P2P_IN: fetch from a peer GPU's HBM
// (a stashed tensor or a peer-homed leaf) — readings E-10, E-11.
enum OpKind : int32_t { OP_H2D = 0, OP_D2H = 1, OP_DROP = 2, OP_CONTRACT = 3, OP_FREE = 4, OP_P2P_OUT = 5, OP_P2P_IN = 6 };
struct LogicalOp { int32_t kind; int32_t node; };

// Capacity-limited LRU plan, readings E-1..E-8.
struct LruPlan {
  std::vector<LogicalOp> ops;
  std::vector<int64_t> used;         // device bytes after each contraction's releases
  int64_t evictions = 0, h2d_count = 0, d2h_count = 0, h2d_bytes = 0, d2h_bytes = 0;
  int64_t peak = 0, transient_peak = 0, host_peak = 0;
  int64_t p2p_out_count = 0, p2p_out_bytes = 0, p2p_in_count = 0, p2p_in_bytes = 0, peer_peak = 0;
};
enum EvictPolicy { EVICT_LRU = 0, EVICT_NEXT_USE = 1 };
// peer_cap: bytes of the peer-HBM eviction tier (E-10; 0: none); peer_home[u] != 0: leaf u's
// home copy is in a peer GPU's HBM (E-11; nullptr: none).
LruPlan lru_plan(const Dag& g, const std::vector<int32_t>& order, int64_t cap, EvictPolicy policy = EVICT_LRU,
                 int64_t peer_cap = 0, const std::vector<uint8_t>* peer_home = nullptr);

// Allocator with coalescing over [0, capacity).  BEST_FIT packs tightly; NEXT_FIT takes
// the first block that fits at or after a rotating cursor (wrapping once), so freed memory
// is reused in FIFO order — the write-after-read distance between a tensor's last reader
// and the next writer of its bytes is as long as the pool allows (more overlap for the
// dataflow executor), at the cost of a higher physical high-water mark.
class RangeAlloc {
 public:
  enum Policy { BEST_FIT = 0, NEXT_FIT = 1 };
  explicit RangeAlloc(int64_t capacity = 0, Policy policy = BEST_FIT);
  int64_t alloc(int64_t bytes);      // -1 if no block fits
  void free(int64_t off, int64_t bytes);
  // allocate exactly [off, off + bytes) if it lies inside one free block; false otherwise
  bool take_range(int64_t off, int64_t bytes);
  const std::map<int64_t, int64_t>& free_blocks() const { return by_off_; }   // offset -> size
  int64_t free_bytes() const;
  int64_t high_water() const { return high_; }
 private:
  std::map<int64_t, int64_t> by_off_;
  std::set<std::pair<int64_t, int64_t>> by_size_;
  int64_t high_ = 0;
  Policy policy_ = BEST_FIT;
  int64_t cursor_ = 0;
  int64_t take(int64_t off, int64_t size, int64_t bytes);
};

// Per-byte-range record of the last op that touched it on each stream, used to derive
// WAR / WAW dependencies when a range is reused (offline, at plan time).
class RangeTracker {
 public:
  explicit RangeTracker(int64_t capacity = 0);
  // ops that a new access by `op` on `stream` must wait for (other streams only)
  void access(int64_t off, int64_t bytes, int stream, int32_t op, std::vector<int32_t>& deps,
              std::vector<int32_t>* same = nullptr);
 private:
  struct Piece { int64_t end; int32_t last[3]; };
  std::map<int64_t, Piece> pieces_;
  void split(int64_t at);
};

enum Stream : int32_t { S_COMPUTE = 0, S_H2D = 1, S_D2H = 2, S_NONE = -1 };

// Where an operand lives at a given op.
enum Loc : int32_t { LOC_POOL = 0, LOC_DEVLEAF = 1, LOC_ROOTS = 2 };

// Compaction move (physical only: the logical plan is unchanged): before the op that needs the
// space, resident tensor `node` is copied device-to-device from src to dst (non-overlapping).
struct Move {
  int32_t node;
  int64_t src, dst, bytes;
};

struct PhysOp {
  int32_t kind;                      // OpKind
  int32_t node;
  int32_t stream;                    // Stream (S_NONE: bookkeeping only)
  int64_t bytes = 0;
  int64_t dev_off = -1;              // pool offset of the tensor this op moves / produces
  int64_t host_off = -1;             // host-pool offset (evicted intermediates), -1: caller leaf
  int64_t peer_off = -1;             // peer-tier offset (P2P_OUT / P2P_IN of a stashed tensor),
                                     // -1: a peer-homed leaf (P2P_IN from the caller's peer copy)
  int32_t loc_a = LOC_POOL, loc_b = LOC_POOL;
  int64_t off_a = -1, off_b = -1;    // operand pool offsets (CONTRACT)
  std::vector<int32_t> deps;         // ops on other streams that must complete first
  std::vector<int32_t> same_deps;    // H2D ops: earlier H2D ops it depends on (implicit in a single
                                     // H2D stream; explicit when H2D copies use several streams)
  bool source = false;               // some later op waits on this one (record an event)
  std::vector<Move> pre_moves;       // compaction moves issued on this op's stream before it
};

struct PhysPlan {
  std::vector<PhysOp> ops;
  int64_t pool_high_water = 0, host_pool_bytes = 0, peer_high_water = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0, p2p_in_bytes = 0, p2p_out_bytes = 0;   // bytes physically copied
  int64_t n_moves = 0, move_bytes = 0;   // compaction (device-to-device) moves
};
// leaf_on_device[u]: the leaf is a caller device buffer (no copy / no pool space).
// peer_bytes: size of the peer-tier region P2P_OUT copies are placed in (best fit;
// CC_E_NOMEM when fragmentation leaves no block).
// compact: when no free block fits an allocation, compact instead of failing — pick the window
// of the needed size whose resident tensors (each at most half the request) are fewest bytes,
// move them device-to-device into free blocks outside it (PhysOp::pre_moves, issued on the
// allocating op's stream with their own dependencies) and allocate the window; CC_E_NOMEM only
// when no window can be cleared.
// leaf_slots: every host leaf gets a fixed slot at the top of the pool (in first-load order) and
// the intermediates share the rest, so no leaf copy ever waits for memory to be freed — the copy
// streams can run ahead at full PCIe rate (useful when the pool holds all leaves next to the
// plan's intermediates; CC_E_NOMEM otherwise, and the caller falls back).
PhysPlan build_phys(const Dag& g, const LruPlan& lp, const std::vector<uint8_t>& leaf_on_device,
                    int64_t pool_bytes, int64_t align, RangeAlloc::Policy policy = RangeAlloc::BEST_FIT,
                    int64_t peer_bytes = 0, bool leaf_slots = false, bool compact = false);

}  // namespace cc
