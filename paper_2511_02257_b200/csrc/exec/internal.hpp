// Executor internals shared by the exec/ translation units (not part of the C ABI).
//
// The executor replays the offline physical plan (host/plan.cpp) on three streams:
// H2D copies (leaf loads, re-fetches) and D2H copies (evictions) on two copy
// streams, contractions on the compute stream; cross-stream dependencies enforce RAW on
// data and WAR/WAW on reused pool memory, so copies run ahead of compute as far as the
// plan's logical residency allows (prefetch without changing the plan).
//   phys.cu           scratch layout + physical placement (prepare_phys)
//   exec_dataflow.cu  persistent-worker executor (prepare_dataflow / issue_dataflow)
//   exec_opbyop.cu    one launch per contraction (issue), Ozaki leaf-form cache, kernel-only replays
//   execute.cu        cc_execute's driver (engine choice, graphs, stats)
//   api.cu            the C ABI
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <queue>
#include <set>
#include <unordered_map>
#include <memory>
#include <string>
#include <vector>

#include "../host/dag.hpp"
#include "../host/partition.hpp"
#include "../host/plan.hpp"
#include "../host/sched.hpp"
#include "../kernels/dataflow.hpp"
#include "../kernels/kernels.hpp"
#include "cc.h"

using namespace cc;

#define CC_VERSION "cc-b200 0.2 (sm_100a; FP64 DMMA + TMA; tcgen05 INT8 Ozaki; sibling/tree/RS-GS schedulers; LRU/next-use plan)"

namespace ccx {
// NVTX range for the executor phases (header-only NVTX 3: a no-op unless a tool such as
// nsys / ncu is attached), so a timeline shows schedule / plan / prepare / issue on the host
// next to the copies and the worker on the device.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
// ctx->opt.debug bit 1: host-side phase times of plan preparation / issue on stderr
struct PhaseTimer {
  const char* what;
  bool on;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  PhaseTimer(const char* w, bool enabled) : what(w), on(enabled) {}
  void lap(const char* step) {
    const auto t1 = std::chrono::steady_clock::now();
    if (on) fprintf(stderr, "[cc timing] %s/%s %.3f ms\n", what, step, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};
constexpr int64_t ALIGN = 1024;
// kind index of a GEMM op for the Ozaki form cache (a leaf's form depends on the problem shape)
constexpr int OZ_KINDS = 5;   // MM1, BM1, BB2, BB1, BT2
inline int oz_kind(int op) {
  return op == CC_MM1 ? 0 : op == CC_BM1 ? 1 : op == CC_BB2 ? 2 : op == CC_BB1 ? 3 : 4;
}
constexpr int GEMM_OPS[5] = {CC_MM1, CC_BM1, CC_BB2, CC_BB1, CC_BT2};
constexpr int TRACE_OPS[2] = {CC_TR_MM, CC_BB3};
inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Traces clustered by shared operand: a permutation of 0..n-1 that puts the traces reading the
// operand most of them read first (adjacent, in their original order), then the next such
// operand among the rest, ...; greedy in O(n log n) (ordered set keyed by remaining count and
// first appearance).  opnd(x, w) is operand w (0, 1) of trace x.
template <class F>
std::vector<int32_t> cluster_by_operand(size_t n, F&& opnd) {
  std::unordered_map<const void*, int32_t> id;
  std::vector<int32_t> cnt, first_at, out;
  std::vector<std::vector<int32_t>> users;
  std::vector<std::array<int32_t, 2>> ids(n);
  for (size_t x = 0; x < n; ++x)
    for (int w = 0; w < 2; ++w) {
      auto ins = id.emplace(opnd(x, w), int32_t(cnt.size()));
      if (ins.second) {
        cnt.push_back(0);
        first_at.push_back(int32_t(x));
        users.emplace_back();
      }
      const int32_t o = ins.first->second;
      ids[x][size_t(w)] = o;
      if (w == 0 || ids[x][0] != o) {
        ++cnt[size_t(o)];
        users[size_t(o)].push_back(int32_t(x));
      }
    }
  std::set<std::array<int32_t, 3>> q;   // (-count, first appearance, operand)
  for (size_t o = 0; o < cnt.size(); ++o) q.insert({-cnt[o], first_at[o], int32_t(o)});
  std::vector<uint8_t> taken(n, 0);
  while (!q.empty()) {
    const int32_t best = (*q.begin())[2];
    q.erase(q.begin());
    for (int32_t x : users[size_t(best)]) {
      if (taken[size_t(x)]) continue;
      taken[size_t(x)] = 1;
      out.push_back(x);
      const int32_t other = ids[size_t(x)][0] == best ? ids[size_t(x)][1] : ids[size_t(x)][0];
      if (other == best) continue;
      q.erase({-cnt[size_t(other)], first_at[size_t(other)], other});
      if (--cnt[size_t(other)] > 0) q.insert({-cnt[size_t(other)], first_at[size_t(other)], other});
    }
    cnt[size_t(best)] = 0;
  }
  return out;
}

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(CC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct KindTimes {
  double seconds[CC_N_OPS] = {0};
  int64_t count[CC_N_OPS] = {0};
};
constexpr int64_t DF_CHUNK_RING = 4;   // GEMM ops split in k that may be in flight at once
constexpr int64_t DF_TRACE_RING = 64;  // TR ops that may be in flight at once
}  // namespace ccx
using namespace ccx;

struct cc_ctx {
  int device = -1;
  cc_options opt{0, 1, 1, 1, 1, 5, 0, 0.0, 0, 1, 1, 1};   // cc_set_options (cc.h)
  bool mm1_ozaki = false;     // execute flags bit 6: MM1/BM1/BB2 on the tcgen05 Ozaki engine (op-by-op)
  int pre_n = 0;              // the plan's first pre_n leaf copies were started before the physical plan
  cudaEvent_t ev_precopy = nullptr;
  // Ozaki leaf-form cache: INT8 slices of leaves, split once per execute and shared by every
  // MM1 reading that leaf in the same role, placed in the pool above the plan's high water
  struct {
    std::vector<OzakiForm> form[2 * OZ_KINDS];   // [2 * oz_kind + (B-form)]
    std::vector<char> have[2 * OZ_KINDS];
    int64_t off = 0, end = 0;
  } oz;
  char* oz_scratch = nullptr;          // reserved leaf-form cache (scratch), may be empty
  int64_t oz_scratch_bytes = 0;
  bool host_only = true;
  char* arena = nullptr;
  int64_t arena_bytes = 0;
  cudaStream_t cs = nullptr, hs = nullptr, ds = nullptr;
  bool own_streams = false;
  int num_sms = 148;
  std::string err;

  Input input;
  bool loaded = false;
  int32_t n_parts = 1, part = 0, mode = 0, t0 = 0, t1 = 0;
  int32_t n_time_parts = 1;            // GRID (mode 2): n_parts TREES parts x n_time_parts TIME parts
  std::vector<int64_t> part_trees;
  std::unique_ptr<Dag> dag;

  bool scheduled = false;
  std::vector<int32_t> order, tree_order;
  ModelTrace mt;
  LruPlan lp;
  cc_plan_stats stats{};
  int64_t cap = 0;

  std::vector<const void*> leaf_host, leaf_dev;
  std::vector<const void*> leaf_peer;   // peer-homed leaves' device copies (E-11), cc_set_leaf_peer
  std::vector<uint8_t> peer_home;       // leaves the current plan fetches from a peer (E-11)
  char* peer_tier = nullptr;            // peer-HBM eviction tier region (E-10), cc_set_peer_tier
  int64_t peer_tier_bytes = 0;

  // physical state
  bool phys_valid = false;
  PhysPlan phys_probe;                  // cc_phys_plan (host-side placement query)
  PhysPlan pp;
  int64_t pool_bytes = 0;
  char* scratch = nullptr;
  size_t gemm_ws_bytes = 0;
  char* gemm_ws = nullptr;
  char* trace_ws = nullptr;
  double2* roots = nullptr;
  double2* corr = nullptr;
  int32_t* term_start = nullptr;
  int32_t* term_tree = nullptr;
  double* term_coef = nullptr;
  std::vector<int32_t> corr_slot_of_term;
  char* host_pool = nullptr;
  int64_t host_pool_bytes = 0;
  std::vector<cudaEvent_t> events;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_h_end = nullptr, ev_d_end = nullptr;
  cudaEvent_t ev_copy_h = nullptr, ev_copy_d = nullptr;   // timing: last copy done (stream mode)
  bool copy_timed = false;
  cudaGraphExec_t gexec = nullptr;
  // kernel-only replays (flags 4: GEMM kinds, 8: TR_MM): the plan's contraction launches of
  // those kinds alone, in plan order, as a CUDA graph -> average launch duration of a kind
  // with no host launch overhead (the roofline measurement)
  cudaGraphExec_t gexec_kind[2] = {nullptr, nullptr};
  bool executed = false;
  KindTimes ktimes;
  int64_t last_n_kernels = 0;
  // plan copies counted as they are enqueued (cc_exec_stats h2d/d2h: runtime counts, not the
  // plan's): the current execute's, and those baked into each cached graph
  int64_t run_h2d = 0, run_d2h = 0, run_p2p_in = 0, run_p2p_out = 0, run_moves = 0;
  int64_t graph_h2d = 0, graph_d2h = 0, graph_p2p_in = 0, graph_p2p_out = 0, graph_moves = 0;   // gexec (op-by-op graph)
  void count_copy(bool h2d, int64_t bytes) { (h2d ? run_h2d : run_d2h) += bytes; }
  // a plan copy of kind OP_H2D / OP_D2H / OP_P2P_IN / OP_P2P_OUT, counted as enqueued
  void count_op_copy(int32_t kind, int64_t bytes) {
    if (kind == OP_P2P_IN) run_p2p_in += bytes;
    else if (kind == OP_P2P_OUT) run_p2p_out += bytes;
    else count_copy(kind == OP_H2D, bytes);
  }

  // dataflow execution (persistent workers): device metadata + per-launch sync area
  bool df_valid = false;
  bool df_slice_major = false;      // the current dataflow queues are in slice-major item order
  char* df_meta = nullptr;          // ops, deps, tensor maps, sync area: top of the pool, else cudaMalloc
  bool df_meta_owned = false;       // cudaMalloc'ed (the arena had no room above the plan's high water)
  char* df_fpart = nullptr;         // fused-trace partials (below the metadata, else cudaMalloc)
  bool df_fpart_owned = false;
  int32_t df_n_fused = 0;
  size_t df_meta_bytes = 0;
  DfArgs df_gemm{};                 // the dataflow worker's arguments (both queues)
  int* df_sync = nullptr;           // zeroed per launch (with the two queue heads before it)
  size_t df_sync_bytes = 0;
  char* df_chunk_ws = nullptr;      // arena scratch: chunk partial rings, trace partial rings
  int64_t df_chunk_slot = 0, df_chunk_cnt_slot = 0;
  char* df_trace_ws = nullptr;
  int64_t df_trace_slot = 0;
  struct DfCopy {
    int32_t op;                     // plan op index
    int32_t stream;                 // S_H2D / S_D2H
    void* dst;
    const void* src;
    size_t bytes;
    int32_t flag_slot;
    std::vector<std::pair<int32_t, int32_t>> wait_values;  // (sync slot, target)
    std::vector<int32_t> wait_events;                        // copy ops on the other copy stream
    bool source = false;
    int32_t chunks = 1;             // H2D in time-slice chunks: the flag counts finished chunks
  };
  std::vector<DfCopy> df_copies;
  std::vector<int32_t> df_issue;    // enqueue order of df_copies (sources before waiters)
  std::vector<uint8_t> df_early;    // per plan op: H2D already enqueued during preparation
  bool df_early_active = false;     // the next issue skips those copies and the sync zeroing
  char* df_sync_base = nullptr;     // queue heads (16 B) + sync ints: top of the pool
  char* df_meta_img = nullptr;      // pinned host image of the dataflow metadata (SM-driven upload)
  size_t df_meta_img_bytes = 0;
  cudaEvent_t ev_meta = nullptr;    // after the last metadata upload (the image is reused)
  std::vector<std::vector<char>> upload_keep;   // host images of prepare_phys uploads
  cudaEvent_t ev_pre = nullptr;
  std::vector<cudaEvent_t> df_events;  // per copy (index into df_copies), when some copy waits on it
  cudaGraphExec_t gexec_df = nullptr;
  int64_t df_gemm_items = 0, df_trace_items = 0;
  unsigned long long* df_prof = nullptr;   // per-item timeline (flags bit 5)

  // direct kernel entry points (GEMM split-K partials; trace partials + zeroed counters)
  char* direct_ws = nullptr;
  size_t direct_ws_bytes = 0;
  char* direct_tr_ws = nullptr;
  size_t direct_tr_ws_bytes = 0;

  ~cc_ctx() { release_device(); }

  void release_df() {
    if (df_prof) cudaFree(df_prof);
    df_prof = nullptr;
    if (gexec_df) cudaGraphExecDestroy(gexec_df);
    gexec_df = nullptr;
    if (df_meta && df_meta_owned) cudaFree(df_meta);
    df_meta = nullptr;
    df_meta_owned = false;
    if (df_fpart && df_fpart_owned) cudaFree(df_fpart);
    df_fpart = nullptr;
    df_fpart_owned = false;
    df_n_fused = 0;
    for (auto e : df_events)
      if (e) cudaEventDestroy(e);
    df_events.clear();
    df_copies.clear();
    df_issue.clear();
    df_valid = false;
  }
  void release_graph() {
    release_df();
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    for (auto& gk : gexec_kind) {
      if (gk) cudaGraphExecDestroy(gk);
      gk = nullptr;
    }
  }
  void release_phys() {
    release_graph();
    release_df();
    for (auto e : events)
      if (e) cudaEventDestroy(e);
    events.clear();
    if (host_pool) cudaFreeHost(host_pool);
    host_pool = nullptr;
    host_pool_bytes = 0;
    phys_valid = false;
  }
  void release_device() {
    if (host_only) return;
    release_phys();
    for (cudaEvent_t* e : {&ev_start, &ev_end, &ev_h_end, &ev_d_end, &ev_copy_h, &ev_copy_d, &ev_pre, &ev_meta,
                           &ev_precopy})
      if (*e) {
        cudaEventDestroy(*e);
        *e = nullptr;
      }
    if (direct_ws) cudaFree(direct_ws);
    direct_ws = nullptr;
    if (df_meta_img) cudaFreeHost(df_meta_img);
    df_meta_img = nullptr;
    df_meta_img_bytes = 0;
    if (direct_tr_ws) cudaFree(direct_tr_ws);
    direct_tr_ws = nullptr;
    if (own_streams) {
      for (cudaStream_t s : {cs, hs, ds})
        if (s) cudaStreamDestroy(s);
    }
    cs = hs = ds = nullptr;
  }
  void need_device() const {
    if (host_only) throw Error(CC_E_STATE, "host-only context (device < 0)");
  }
};

namespace ccx {
void rebuild_dag(cc_ctx* ctx);
ZgemmProblem problem_for(int op, int64_t Lt, int64_t N, int64_t S, const void* a, const void* b, void* c);
void df_gemm_geometry(const ZgemmProblem& p, int64_t& tiles, int64_t& KT, int64_t& chunks, int num_sms);
int64_t df_trace_pieces(const TraceShape& sh);
struct ScratchSizes {
  int64_t sz_gemm = 0, sz_trace = 0, sz_roots = 0, sz_corr = 0, sz_ts = 0, sz_tt = 0, sz_tc = 0, sz_df_chunk = 0,
          sz_df_trace = 0, sz_ozc = 0, total = 0;
};
ScratchSizes scratch_sizes(cc_ctx* ctx);
void prepare_phys(cc_ctx* ctx);
void prepare_dataflow(cc_ctx* ctx, bool early = false);
int issue_dataflow(cc_ctx* ctx, bool time_copies = false);
void oz_cache_reset(cc_ctx* ctx);
int issue(cc_ctx* ctx, bool time_kernels, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* kev,
          std::vector<int>* kev_kind);
void kernel_only(cc_ctx* ctx, int cls, cc_exec_stats* stats);
void execute(cc_ctx* ctx, int32_t flags, bool blocking, cc_exec_stats* stats);
// Source of a P2P_IN of a peer-homed leaf (E-11): this part's time slices of the caller's copy.
inline const void* peer_leaf_src(cc_ctx* ctx, int32_t u) {
  const Dag& g = *ctx->dag;
  const Node& n = g.nodes[size_t(u)];
  const char* p = static_cast<const char*>(ctx->leaf_peer[size_t(u)]);
  if (!p) throw Error(CC_E_STATE, "leaf " + std::to_string(n.id) + " has no peer copy (cc_set_leaf_peer)");
  const int64_t per_t_m = 16LL * g.N * g.N;
  const int64_t per_t = n.op == CC_LEAF_M ? per_t_m : per_t_m * g.S * g.N;
  return p + int64_t(ctx->t0) * per_t;
}
}  // namespace ccx

