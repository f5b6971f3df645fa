// C ABI (include/cc.h) and the device executor.
//
// The executor replays the offline physical plan (host/plan.cpp) on three streams:
// H2D copies (leaf loads, re-fetches) and D2H copies (evictions) on two copy
// streams, contractions on the compute stream; cross-stream event edges enforce RAW on
// data and WAR/WAW on reused pool memory, so copies run ahead of compute as far as the
// plan's logical residency allows (prefetch without changing the plan).  The whole
// replay can be captured once as a CUDA graph and relaunched.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <queue>
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

namespace {
// CC_TIMING=1: host-side phase times of plan preparation / issue on stderr
struct PhaseTimer {
  const char* what;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit PhaseTimer(const char* w) : what(w) {}
  void lap(const char* step) {
    static const bool on = getenv("CC_TIMING") != nullptr;
    const auto t1 = std::chrono::steady_clock::now();
    if (on) fprintf(stderr, "[cc timing] %s/%s %.3f ms\n", what, step, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};
}  // namespace

#define CC_VERSION "cc-b200 0.1 (sm_100a; FP64 DMMA + TMA; sibling/tree schedulers; LRU plan)"

namespace {

constexpr int64_t ALIGN = 1024;
// INT8 slices per operand of the Ozaki MM1 engine (reading V-6: 5 balanced base-256 digits,
// 38 bits; phase-limited MM1 errors <= 1e-11 relative in the tests, inside the 1e-10 bar).
constexpr int OZAKI_SLICES = 5;
// kind index of a GEMM op for the Ozaki form cache (a leaf's form depends on the problem shape)
inline int oz_kind(int op) { return op == CC_MM1 ? 0 : (op == CC_BM1 ? 1 : 2); }
int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(CC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct KindTimes {
  double seconds[8] = {0};
  int64_t count[8] = {0};
};

}  // namespace

struct cc_ctx {
  int device = -1;
  bool mm1_ozaki = false;     // execute flags bit 6: MM1/BM1/BB2 on the tcgen05 Ozaki engine (op-by-op)
  int pre_n = 0;              // the plan's first pre_n leaf copies were started before the physical plan
  cudaEvent_t ev_precopy = nullptr;
  // Ozaki leaf-form cache: INT8 slices of leaves, split once per execute and shared by every
  // MM1 reading that leaf in the same role, placed in the pool above the plan's high water
  struct {
    std::vector<OzakiForm> form[6];   // [2 * oz_kind + (B-form)]
    std::vector<char> have[6];
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
  std::vector<int64_t> part_trees;
  std::unique_ptr<Dag> dag;

  bool scheduled = false;
  std::vector<int32_t> order, tree_order;
  ModelTrace mt;
  LruPlan lp;
  cc_plan_stats stats{};
  int64_t cap = 0;

  std::vector<const void*> leaf_host, leaf_dev;

  // physical state
  bool phys_valid = false;
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

  // dataflow execution (persistent workers): device metadata + per-launch sync area
  bool df_valid = false;
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
  cudaStream_t cs2 = nullptr;       // second compute stream (trace worker)
  cudaEvent_t ev_cs2 = nullptr;
  cudaStream_t hs2 = nullptr;       // second H2D stream: wait-free leaf copies alternate with hs
  cudaEvent_t ev_hs2 = nullptr;
  cudaStream_t hsx[3] = {nullptr, nullptr, nullptr};   // op-by-op: extra H2D streams
  cudaEvent_t ev_hsx[3] = {nullptr, nullptr, nullptr};
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
    if (cs2) cudaStreamDestroy(cs2);
    cs2 = nullptr;
    if (hs2) cudaStreamDestroy(hs2);
    hs2 = nullptr;
    for (int k = 0; k < 3; ++k) {
      if (hsx[k]) cudaStreamDestroy(hsx[k]);
      if (ev_hsx[k]) cudaEventDestroy(ev_hsx[k]);
      hsx[k] = nullptr;
      ev_hsx[k] = nullptr;
    }
    if (ev_hs2) cudaEventDestroy(ev_hs2);
    ev_hs2 = nullptr;
    if (ev_cs2) cudaEventDestroy(ev_cs2);
    ev_cs2 = nullptr;
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

static cc_status fail(cc_ctx* ctx, const Error& e) {
  if (ctx) ctx->err = e.what();
  return e.status;
}

#define API_BEGIN try {
#define API_END                                                   \
  }                                                               \
  catch (const Error& e) { return fail(ctx, e); }                 \
  catch (const std::bad_alloc&) {                                 \
    if (ctx) ctx->err = "host allocation failed";                 \
    return CC_E_NOMEM;                                            \
  }                                                               \
  catch (const std::exception& e) {                               \
    if (ctx) ctx->err = e.what();                                 \
    return CC_E_INVAL;                                            \
  }                                                               \
  return CC_OK;

// ------------------------------------------------------------------------------------------
namespace {

void rebuild_dag(cc_ctx* ctx) {
  const int32_t Lt = ctx->input.dims.Lt;
  if (ctx->n_parts <= 1) {
    ctx->t0 = 0;
    ctx->t1 = Lt;
    ctx->dag = std::make_unique<Dag>(ctx->input);
    ctx->part_trees.clear();
    for (const auto& t : ctx->dag->trees) ctx->part_trees.push_back(t.tree_id);
  } else if (ctx->mode == 0) {
    ctx->t0 = int32_t(int64_t(ctx->part) * Lt / ctx->n_parts);
    ctx->t1 = int32_t(int64_t(ctx->part + 1) * Lt / ctx->n_parts);
    if (ctx->t1 <= ctx->t0) throw Error(CC_E_INVAL, "TIME partition: part has no time slices");
    ctx->dag = std::make_unique<Dag>(ctx->input, ctx->t1 - ctx->t0);
    ctx->part_trees.clear();
    for (const auto& t : ctx->dag->trees) ctx->part_trees.push_back(t.tree_id);
  } else {
    ctx->t0 = 0;
    ctx->t1 = Lt;
    Dag full(ctx->input);
    std::vector<int32_t> parts = tree_parts(full, ctx->n_parts, nullptr);
    std::vector<int64_t> keep;
    for (size_t t = 0; t < full.trees.size(); ++t)
      if (parts[t] == ctx->part) keep.push_back(full.trees[t].tree_id);
    if (keep.empty()) throw Error(CC_E_INVAL, "TREES partition: part has no trees");
    ctx->dag = std::make_unique<Dag>(ctx->input, 0, &keep);
    ctx->part_trees = keep;
  }
  const size_t n = ctx->dag->nodes.size();
  ctx->leaf_host.assign(n, nullptr);
  ctx->leaf_dev.assign(n, nullptr);
  ctx->scheduled = false;
  ctx->executed = false;
  ctx->phys_valid = false;
  ctx->release_graph();
}

ZgemmProblem problem_for(int op, int64_t Lt, int64_t N, int64_t S, const void* a, const void* b, void* c) {
  ZgemmProblem p{};
  p.A = a;
  p.B = b;
  p.C = c;
  p.batch = Lt;
  if (op == CC_MM1) {
    p.M = N; p.Nn = N; p.Kin = N; p.Ko = 1;
    p.lda = N; p.sAo = 0; p.sAb = N * N;
    p.ldb = N; p.sBo = 0; p.sBb = N * N;
    p.ldc = N; p.sCb = N * N;
  } else if (op == CC_BM1) {
    p.M = S * N * N; p.Nn = N; p.Kin = N; p.Ko = 1;
    p.lda = N; p.sAo = 0; p.sAb = S * N * N * N;
    p.ldb = N; p.sBo = 0; p.sBb = N * N;
    p.ldc = N; p.sCb = S * N * N * N;
  } else {  // CC_BB2
    p.M = N; p.Nn = N; p.Kin = N * N; p.Ko = S;
    p.lda = N * N; p.sAo = N * N * N; p.sAb = S * N * N * N;
    p.ldb = N; p.sBo = N * N * N; p.sBb = S * N * N * N;
    p.ldc = N; p.sCb = N * N;
  }
  return p;
}

constexpr int64_t DF_CHUNK_RING = 4;   // GEMM ops split in k that may be in flight at once
constexpr int64_t DF_TRACE_RING = 16;  // TR ops that may be in flight at once

// Work split of one GEMM op for the dataflow worker: tiles of BM x BN, KT k-tiles; an op
// with fewer tiles than SMs is split into k-chunks so it still spreads over the GPU.
void df_gemm_geometry(const ZgemmProblem& p, int64_t& tiles, int64_t& KT, int64_t& chunks, int num_sms) {
  int BM, BN, BK, slot;
  df_gemm_tile_dims(&BM, &BN, &BK, &slot);
  tiles = ((p.M + BM - 1) / BM) * ((p.Nn + BN - 1) / BN) * p.batch;
  KT = p.Ko * ((p.Kin + BK - 1) / BK);
  chunks = 1;
  if (tiles < num_sms) {
    const int64_t want = (2 * num_sms + tiles - 1) / tiles;
    const int64_t cap = std::max<int64_t>(1, KT / 4);
    chunks = std::min(want, cap);
  }
}

// Pieces per time slice of a TR op: ~DF_TR_UNITS blocks of 32x32 (32 KB each) per item.
int64_t df_trace_pieces(int64_t Lt, int64_t N) {
  static const int64_t units = getenv("CC_DF_TR_UNITS") ? std::max(1LL, atoll(getenv("CC_DF_TR_UNITS"))) : 16;
  const int64_t nb = (N + 31) / 32, U = nb * nb;
  (void)Lt;
  return std::max<int64_t>(1, (U + units - 1) / units);
}

// Sets up scratch (kernel workspace, roots, correlators, term tables), the physical plan,
// events and the host pool.  Called lazily by cc_execute.
void prepare_phys(cc_ctx* ctx) {
  if (ctx->phys_valid) return;
  PhaseTimer pt("prepare_phys");
  ctx->release_phys();
  pt.lap("release");
  const Dag& g = *ctx->dag;
  if (g.abstract) throw Error(CC_E_STATE, "abstract DAG (leafX/OPX) can be scheduled, not executed");
  const int64_t Lt = g.Lt, N = g.N, S = g.S;
  // scratch layout
  size_t gemm_ws = 0;
  bool has[8] = {false};
  for (const auto& n : g.nodes) has[n.op] = true;
  for (int op : {int(CC_MM1), int(CC_BM1), int(CC_BB2)})
    if (has[op]) gemm_ws = std::max(gemm_ws, zgemm_workspace_bytes(problem_for(op, Lt, N, S, nullptr, nullptr, nullptr), ctx->num_sms));
  // Ozaki engine (execute flags bit 6): workspace for batches of time slices that fit in
  // max(one slice, arena / 16)
  for (int op : {int(CC_MM1), int(CC_BM1), int(CC_BB2)}) {
    if (!has[op]) continue;
    const ZgemmProblem q = problem_for(op, Lt, N, S, nullptr, nullptr, nullptr);
    const size_t lim = std::max(ozaki_workspace_bytes(q, OZAKI_SLICES, 1), size_t(ctx->arena_bytes / 16));
    int64_t bt = Lt;
    while (bt > 1 && ozaki_workspace_bytes(q, OZAKI_SLICES, bt) > lim) bt = (bt + 1) / 2;
    gemm_ws = std::max(gemm_ws, ozaki_workspace_bytes(q, OZAKI_SLICES, bt));
  }
  // Ozaki leaf-form cache: one form per (leaf, op kind, side) read by a GEMM op; reserved
  // when it takes at most 1/8 of the arena (else the cache uses whatever pool space the plan
  // leaves free)
  int64_t sz_ozc = 0;
  {
    std::vector<std::array<char, 6>> role(g.nodes.size(), std::array<char, 6>{});
    for (const auto& n : g.nodes)
      if (n.op == CC_MM1 || n.op == CC_BM1 || n.op == CC_BB2) {
        if (g.nodes[size_t(n.l)].leaf()) role[size_t(n.l)][size_t(2 * oz_kind(n.op))] = 1;
        if (g.nodes[size_t(n.r)].leaf()) role[size_t(n.r)][size_t(2 * oz_kind(n.op) + 1)] = 1;
      }
    int64_t fsz[6] = {0};
    for (int op : {int(CC_MM1), int(CC_BM1), int(CC_BB2)}) {
      if (!has[op]) continue;
      const ZgemmProblem q = problem_for(op, Lt, N, S, nullptr, nullptr, nullptr);
      fsz[2 * oz_kind(op)] = round_up(int64_t(ozaki_form_bytes(q, OZAKI_SLICES, false)), ALIGN);
      fsz[2 * oz_kind(op) + 1] = round_up(int64_t(ozaki_form_bytes(q, OZAKI_SLICES, true)), ALIGN);
    }
    for (const auto& r : role)
      for (int k = 0; k < 6; ++k) sz_ozc += r[size_t(k)] ? fsz[k] : 0;
    if (sz_ozc > ctx->arena_bytes / 8) sz_ozc = 0;
  }
  const size_t trace_ws = trace_workspace_bytes(Lt, N);
  const int64_t n_trees = int64_t(g.trees.size()), n_corr = int64_t(g.corr_ids.size()), n_terms = int64_t(g.terms.size());
  const int64_t sz_gemm = round_up(int64_t(gemm_ws), ALIGN), sz_trace = round_up(int64_t(trace_ws), ALIGN);
  const int64_t sz_roots = round_up(n_trees * Lt * 16, ALIGN), sz_corr = round_up(std::max<int64_t>(n_corr, 1) * Lt * 16, ALIGN);
  const int64_t sz_ts = round_up((n_corr + 1) * 4, ALIGN), sz_tt = round_up(std::max<int64_t>(n_terms, 1) * 4, ALIGN);
  const int64_t sz_tc = round_up(std::max<int64_t>(n_terms, 1) * 16, ALIGN);
  // dataflow workspaces: rings of chunk-partial slots (GEMM ops split in k) and of trace
  // partial slots (per-op tickets and [Lt][P] partials)
  ctx->df_chunk_slot = ctx->df_chunk_cnt_slot = 0;
  for (int op : {int(CC_MM1), int(CC_BM1), int(CC_BB2)}) {
    if (!has[op]) continue;
    int64_t tiles, KT, chunks;
    df_gemm_geometry(problem_for(op, Lt, N, S, nullptr, nullptr, nullptr), tiles, KT, chunks, ctx->num_sms);
    if (chunks > 1) {
      int BM, BN, BK, slot;
      df_gemm_tile_dims(&BM, &BN, &BK, &slot);
      ctx->df_chunk_slot = std::max(ctx->df_chunk_slot, round_up(tiles * chunks * slot * 8, ALIGN));
      ctx->df_chunk_cnt_slot = std::max(ctx->df_chunk_cnt_slot, round_up(tiles * 4, ALIGN));
    }
  }
  ctx->df_trace_slot = round_up(Lt * df_trace_pieces(Lt, N) * 16, ALIGN) + round_up(Lt * 4, ALIGN);
  const int64_t sz_df_chunk = DF_CHUNK_RING * (ctx->df_chunk_slot + ctx->df_chunk_cnt_slot);
  const int64_t sz_df_trace = DF_TRACE_RING * ctx->df_trace_slot;
  const int64_t scratch = sz_gemm + sz_trace + sz_roots + sz_corr + sz_ts + sz_tt + sz_tc + sz_df_chunk + sz_df_trace + sz_ozc;
  const int64_t pool = (ctx->arena_bytes - scratch) / ALIGN * ALIGN;
  if (pool <= 0) throw Error(CC_E_NOMEM, "arena too small for the kernel workspace (" + std::to_string(scratch) + " B)");
  ctx->pool_bytes = pool;
  char* s = ctx->arena + pool;
  ctx->gemm_ws = s; ctx->gemm_ws_bytes = size_t(sz_gemm); s += sz_gemm;
  ctx->trace_ws = s; s += sz_trace;
  ctx->roots = reinterpret_cast<double2*>(s); s += sz_roots;
  ctx->corr = reinterpret_cast<double2*>(s); s += sz_corr;
  ctx->term_start = reinterpret_cast<int32_t*>(s); s += sz_ts;
  ctx->term_tree = reinterpret_cast<int32_t*>(s); s += sz_tt;
  ctx->term_coef = reinterpret_cast<double*>(s); s += sz_tc;
  ctx->df_chunk_ws = s; s += sz_df_chunk;
  ctx->df_trace_ws = s; s += sz_df_trace;
  ctx->oz_scratch = s; ctx->oz_scratch_bytes = sz_ozc; s += sz_ozc;
  // every upload / clear is ordered on the compute stream (the copy streams may already be
  // busy; a legacy-stream cudaMemcpy from pageable memory can return before its DMA lands)
  if (sz_df_chunk > 0) ck(cudaMemsetAsync(ctx->df_chunk_ws, 0, size_t(sz_df_chunk), ctx->cs), "dataflow workspace");
  if (sz_df_trace > 0) ck(cudaMemsetAsync(ctx->df_trace_ws, 0, size_t(sz_df_trace), ctx->cs), "dataflow workspace");
  // term tables grouped by correlator slot (corr ids ascending), input order within a slot
  std::vector<int32_t> start(size_t(n_corr) + 1, 0), tree(size_t(std::max<int64_t>(n_terms, 1)), 0);
  std::vector<double> coef(size_t(std::max<int64_t>(n_terms, 1)) * 2, 0.0);
  {
    std::vector<int32_t> slot(static_cast<size_t>(n_terms));
    for (int64_t k = 0; k < n_terms; ++k) {
      const auto it = std::lower_bound(g.corr_ids.begin(), g.corr_ids.end(), g.terms[size_t(k)].corr_id);
      slot[size_t(k)] = int32_t(it - g.corr_ids.begin());
      ++start[size_t(slot[size_t(k)]) + 1];
    }
    for (int64_t c = 0; c < n_corr; ++c) start[size_t(c) + 1] += start[size_t(c)];
    std::vector<int32_t> fill(start.begin(), start.end() - 1);
    for (int64_t k = 0; k < n_terms; ++k) {
      const int32_t pos = fill[size_t(slot[size_t(k)])]++;
      tree[size_t(pos)] = g.terms[size_t(k)].tree;
      coef[2 * size_t(pos)] = g.terms[size_t(k)].coef.real();
      coef[2 * size_t(pos) + 1] = g.terms[size_t(k)].coef.imag();
    }
  }
  ctx->upload_keep.clear();
  auto upload = [&](void* dst, std::vector<char>&& img) {
    ctx->upload_keep.push_back(std::move(img));   // host image alive until the next prepare
    const auto& v = ctx->upload_keep.back();
    ck(cudaMemcpyAsync(dst, v.data(), v.size(), cudaMemcpyHostToDevice, ctx->cs), "upload");
  };
  auto bytes_of = [](const auto& vec) {
    const char* p = reinterpret_cast<const char*>(vec.data());
    return std::vector<char>(p, p + vec.size() * sizeof(vec[0]));
  };
  upload(ctx->term_start, bytes_of(start));
  upload(ctx->term_tree, bytes_of(tree));
  upload(ctx->term_coef, bytes_of(coef));
  ck(cudaMemsetAsync(ctx->trace_ws, 0, trace_ws, ctx->cs), "trace counters");
  if (sz_gemm > 0) ck(cudaMemsetAsync(ctx->gemm_ws, 0, size_t(sz_gemm), ctx->cs), "gemm flags");
  ck(cudaMemsetAsync(ctx->roots, 0, size_t(sz_roots), ctx->cs), "roots");
  pt.lap("scratch+tables");
  // physical plan over the pool
  std::vector<uint8_t> on_dev(g.nodes.size(), 0);
  for (size_t u = 0; u < g.nodes.size(); ++u) on_dev[u] = ctx->leaf_dev[u] != nullptr;
  // Placement: next-fit over the pool (freed memory is reused in FIFO order, so the next
  // writer of a byte range rarely has to wait for its last reader — the dataflow executor
  // overlaps more).  With a capacity cap the physical pool is held to 1.25 x cap so the
  // physical footprint follows the logical one; the logical plan is unchanged either way.
  // (CC_PHYS_SLACK: the slack fraction over the cap, default 0.25)
  int64_t phys_limit = pool;
  static const double slack = getenv("CC_PHYS_SLACK") ? atof(getenv("CC_PHYS_SLACK")) : 0.25;
  if (ctx->cap > 0) phys_limit = std::min(pool, round_up(ctx->cap + int64_t(double(ctx->cap) * slack), ALIGN));
  try {
    ctx->pp = build_phys(g, ctx->lp, on_dev, phys_limit, ALIGN, RangeAlloc::NEXT_FIT);
  } catch (const Error& e) {
    if (e.status != CC_E_NOMEM) throw;
    ctx->pp = build_phys(g, ctx->lp, on_dev, pool, ALIGN, RangeAlloc::BEST_FIT);
  }
  ctx->stats.arena_high_water = ctx->pp.pool_high_water;
  pt.lap("build_phys");
  if (ctx->pp.host_pool_bytes > 0) {
    ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->host_pool), size_t(ctx->pp.host_pool_bytes), cudaHostAllocDefault),
       "pinned host pool");
    ctx->host_pool_bytes = ctx->pp.host_pool_bytes;
  }
  ctx->events.assign(ctx->pp.ops.size(), nullptr);
  for (size_t i = 0; i < ctx->pp.ops.size(); ++i)
    if (ctx->pp.ops[i].source) ck(cudaEventCreateWithFlags(&ctx->events[i], cudaEventDisableTiming), "event");
  pt.lap("host pool+events");
  ctx->phys_valid = true;
}


// ------------------------------------------------------------------------------------------
// Dataflow execution: the plan's contractions as work items of two persistent workers,
// copies on the copy streams, synchronised through integer slots (kernels/dataflow.hpp).

// Reads/writes of byte ranges in plan order -> data dependencies between plan ops (RAW on the
// last writer; WAR/WAW on the last writer and every reader since).
class RWTracker {
 public:
  explicit RWTracker(int64_t capacity) { pieces_[0] = Piece{std::max<int64_t>(capacity, 1), -1, {}}; }
  void read(int64_t off, int64_t n, int32_t op, std::vector<int32_t>& deps) {
    visit(off, n, [&](Piece& p) {
      if (p.writer >= 0) deps.push_back(p.writer);
      p.readers.push_back(op);
    });
  }
  // the latest writer of any byte in [off, off+n) (-1: never written)
  int32_t last_writer(int64_t off, int64_t n) {
    int32_t w = -1;
    visit(off, n, [&](Piece& p) { w = std::max(w, p.writer); });
    return w;
  }
  void write(int64_t off, int64_t n, int32_t op, std::vector<int32_t>& deps) {
    visit(off, n, [&](Piece& p) {
      if (p.writer >= 0) deps.push_back(p.writer);
      deps.insert(deps.end(), p.readers.begin(), p.readers.end());
      p.readers.clear();
      p.writer = op;
    });
  }

 private:
  struct Piece {
    int64_t end;
    int32_t writer;
    std::vector<int32_t> readers;
  };
  std::map<int64_t, Piece> pieces_;
  void split(int64_t at) {
    auto it = pieces_.upper_bound(at);
    if (it == pieces_.begin()) return;
    --it;
    if (it->first == at || it->second.end <= at) return;
    Piece hi = it->second;
    it->second.end = at;
    pieces_[at] = hi;
  }
  template <class F>
  void visit(int64_t off, int64_t n, F f) {
    split(off);
    split(off + n);
    for (auto it = pieces_.find(off); it != pieces_.end() && it->first < off + n; ++it) f(it->second);
  }
};

using PFN_waitval = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitval df_wait_fn() {
  static PFN_waitval fn = nullptr;
  static bool done = false;
  if (!done) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitval>(p);
    done = true;
  }
  return fn;
}
PFN_waitval df_write_fn() {
  static PFN_waitval fn = nullptr;
  static bool done = false;
  if (!done) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitval>(p);
    done = true;
  }
  return fn;
}

// Source / destination of a plan copy op.
std::pair<const void*, void*> copy_endpoints(cc_ctx* ctx, const PhysOp& op) {
  const Dag& g = *ctx->dag;
  const Node& n = g.nodes[size_t(op.node)];
  if (op.kind == OP_H2D) {
    if (n.leaf()) {
      const char* h = static_cast<const char*>(ctx->leaf_host[size_t(op.node)]);
      if (!h) throw Error(CC_E_STATE, "leaf " + std::to_string(n.id) + " has no data (cc_set_leaf)");
      const int64_t per_t_m = 16LL * g.N * g.N;
      const int64_t per_t = n.op == CC_LEAF_M ? per_t_m : per_t_m * g.S * g.N;
      return {h + int64_t(ctx->t0) * per_t, ctx->arena + op.dev_off};
    }
    return {ctx->host_pool + op.host_off, ctx->arena + op.dev_off};
  }
  return {ctx->arena + op.dev_off, ctx->host_pool + op.host_off};
}

// One plan copy on `s`: C time-slice chunks, each followed by a flag write (value = chunks
// done) — the dataflow worker's items wait on the flag (chunk of their slice, kernels/dataflow.hpp).
void enqueue_copy(cc_ctx* ctx, cudaStream_t s, const void* src, void* dst, size_t bytes, cudaMemcpyKind kind,
                  int32_t chunks, int32_t flag_slot) {
  const Dag& g = *ctx->dag;
  const size_t per_t = bytes / size_t(std::max<int64_t>(g.Lt, 1));
  for (int32_t ch = 0; ch < chunks; ++ch) {
    // chunk ch: slices [ch*Lt/C, (ch+1)*Lt/C)
    const size_t t0 = chunks == 1 ? 0 : size_t(int64_t(ch) * g.Lt / chunks);
    const size_t t1 = chunks == 1 ? 0 : size_t(int64_t(ch + 1) * g.Lt / chunks);
    const size_t off = t0 * per_t, len = chunks == 1 ? bytes : (t1 - t0) * per_t;
    ck(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len, kind, s), "copy");
    if (df_write_fn()(s, reinterpret_cast<CUdeviceptr>(ctx->df_sync + flag_slot), cuuint32_t(ch + 1), 0) != CUDA_SUCCESS)
      throw Error(CC_E_CUDA, "cuStreamWriteValue32 failed");
  }
}

// Wait-free H2D copies alternate between the H2D stream and a second one (CC_H2D_STREAMS=1
// keeps one): each copy is followed by its flag write, a stream memory operation that idles
// its stream's copy engine (~8 us measured), so the other stream's copy fills the gap.
// Off by default: 4 alternating c2 runs each: copies land 80 us earlier with two streams but
// e2e is 10.82-10.84 ms vs 10.74-10.75 ms with one (the leaves arrive in a less useful order).
bool dual_h2d() {
  static const int n = getenv("CC_H2D_STREAMS") ? atoi(getenv("CC_H2D_STREAMS")) : 1;
  return n >= 2;
}
void ensure_hs2(cc_ctx* ctx) {
  if (!ctx->hs2) {
    ck(cudaStreamCreateWithFlags(&ctx->hs2, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ctx->ev_hs2, cudaEventDisableTiming), "event");
  }
}

// early: start the wait-free H2D copies at the head of the copy order on the H2D stream as
// soon as that order is known, so they overlap the rest of the host-side preparation (queues,
// tensor maps, upload); the next issue_dataflow only adds their flag writes.
void prepare_dataflow(cc_ctx* ctx, bool early = false) {
  if (ctx->df_valid) return;
  if (getenv("CC_DEBUG")) fprintf(stderr, "[cc] prepare_dataflow\n");
  prepare_phys(ctx);
  PhaseTimer tmr("prepare_dataflow");
  const Dag& g = *ctx->dag;
  const auto& ops = ctx->pp.ops;
  const int64_t Lt = g.Lt, N = g.N;
  const int32_t n_ops = int32_t(ops.size());
  const int64_t per_t_m = 16LL * g.N * g.N;
  // sync slots (done counters of compute ops, flags of copies) and H2D chunk counts
  std::vector<int32_t> slot(size_t(n_ops), -1), target(size_t(n_ops), 0), df_index(size_t(n_ops), -1);
  int32_t n_sync = 0;
  // per-time-slice done counters of GEMMs with meson outputs [Lt, N, N] (MM1, BB2): a trace of
  // slice t waits only for that slice's tiles (CC_SLICE_DEPS=0: for the whole GEMM)
  std::vector<int32_t> slice_slot(size_t(n_ops), -1), items_per_slice(size_t(n_ops), 0);
  static const bool slice_deps = !(getenv("CC_SLICE_DEPS") && atoi(getenv("CC_SLICE_DEPS")) == 0);
  // CC_H2D_CHUNK_MB: H2D copies in time-slice chunks of about that size (default off: every
  // chunk costs a stream memory operation, measured ~8 us of copy-engine idle each on B200)
  const double chunk_mb = getenv("CC_H2D_CHUNK_MB") ? atof(getenv("CC_H2D_CHUNK_MB")) : 0.0;
  const int64_t h2d_chunk = chunk_mb > 0 ? std::max<int64_t>(4096, int64_t(chunk_mb * 1048576.0)) : INT64_MAX;
  for (int32_t i = 0; i < n_ops; ++i) {
    const PhysOp& op = ops[size_t(i)];
    if (op.stream == S_NONE) continue;
    slot[size_t(i)] = n_sync++;
    if (slice_deps && op.kind == OP_CONTRACT && Lt > 1 &&
        (g.nodes[size_t(op.node)].op == CC_MM1 || g.nodes[size_t(op.node)].op == CC_BB2)) {
      slice_slot[size_t(i)] = n_sync;
      n_sync += int32_t(Lt);
    }
    if (op.kind != OP_CONTRACT) {
      // consumers of a copy in C > 1 time-slice chunks wait only for the chunk holding their
      // slice (target -C); else the flag reaches 1
      target[size_t(i)] = 1;
      if (op.kind == OP_H2D && op.stream == S_H2D && Lt > 1 && op.bytes % Lt == 0) {
        const int64_t C = std::min<int64_t>(Lt, std::max<int64_t>(1, op.bytes / h2d_chunk + (op.bytes % h2d_chunk != 0)));
        if (C > 1) target[size_t(i)] = -int32_t(C);
      }
    }
  }
  // The sync area (2 queue heads + n_sync ints), zeroed before every launch, sits at the top
  // of the pool (above the plan's high-water mark); the rest of the metadata goes below it.
  const size_t sz_sync = round_up(16 + int64_t(n_sync) * 4, 256);
  {
    const int64_t sync_off = (ctx->pool_bytes - int64_t(sz_sync)) / 256 * 256;
    if (sync_off < ctx->pp.pool_high_water) throw Error(CC_E_NOMEM, "arena too small for the dataflow sync area");
    ctx->df_sync_base = ctx->arena + sync_off;
    ctx->df_sync = reinterpret_cast<int*>(ctx->df_sync_base + 16);
    ctx->df_sync_bytes = sz_sync;
  }
  // 0b. early H2D copies.  A leaf H2D whose device range lies above everything the plan
  // touched before it (fresh pool memory) waits on nothing and nothing earlier depends on it:
  // it may be issued first, before the dependency analysis, so the copy engine starts while
  // the host builds the rest.  These copies are ordered greedily by the work they enable:
  // next = the leaf that completes the leaf set (closure in the DAG) of the most estimated
  // compute time, so the GEMMs — most of the step — start early and little is left once the
  // last leaf lands.  CC_COPY_REORDER=0 keeps plan order.
  std::vector<int32_t> early_seq;
  std::vector<uint8_t> is_early(size_t(n_ops), 0);
  int32_t n_first = 0;                                 // early copies already enqueued (plan ops 0..n-1)
  {
    int64_t touched_end = 0;
    auto touch = [&](int64_t off, int64_t bytes) {
      if (off >= 0) touched_end = std::max(touched_end, off + bytes);
    };
    for (int32_t i = 0; i < n_ops; ++i) {
      const PhysOp& op = ops[size_t(i)];
      const Node& n = g.nodes[size_t(op.node)];
      const int64_t rb = round_up(n.size, ALIGN);
      if (op.kind == OP_H2D && op.stream == S_H2D && n.leaf() && op.dev_off >= touched_end) {
        is_early[size_t(i)] = 1;
        early_seq.push_back(i);
      }
      if (op.kind == OP_H2D || op.kind == OP_D2H) touch(op.dev_off, rb);
      if (op.kind == OP_CONTRACT) {
        if (op.loc_a == LOC_POOL) touch(op.off_a, round_up(g.nodes[size_t(n.l)].size, ALIGN));
        if (op.loc_b == LOC_POOL) touch(op.off_b, round_up(g.nodes[size_t(n.r)].size, ALIGN));
        touch(op.dev_off, rb);
      }
    }
    const int reorder = getenv("CC_COPY_REORDER") ? atoi(getenv("CC_COPY_REORDER")) : 1;
    // the plan's first leaf copies start now, before the ordering of the others is computed
    // (they head the order either way); the first pre_n of them were even started by
    // execute() before the physical plan existed, and only get their flag writes here
    if (early && !early_seq.empty()) {
      ck(cudaEventRecord(ctx->ev_pre, ctx->cs), "event");        // after all earlier work on cs
      ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_pre, 0), "wait");
      ck(cudaMemsetAsync(ctx->df_sync_base, 0, sz_sync, ctx->hs), "memset");
      int pre = ctx->pre_n;
      for (int j = 0; j < pre; ++j)
        if (size_t(j) >= early_seq.size() || early_seq[size_t(j)] != j || target[size_t(j)] != 1) pre = 0;
      if (pre == 0 && ctx->pre_n > 0) ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_precopy, 0), "wait");
      for (int j = 0; j < pre; ++j)   // hs order: copies, memset, flags
        if (df_write_fn()(ctx->hs, reinterpret_cast<CUdeviceptr>(ctx->df_sync + slot[size_t(j)]), 1u, 0) != CUDA_SUCCESS)
          throw Error(CC_E_CUDA, "cuStreamWriteValue32 failed");
      if (pre == 0) {
        const int32_t i = early_seq[0];
        const auto ep = copy_endpoints(ctx, ops[size_t(i)]);
        enqueue_copy(ctx, ctx->hs, ep.first, ep.second, size_t(ops[size_t(i)].bytes), cudaMemcpyHostToDevice,
                     target[size_t(i)] < 0 ? -target[size_t(i)] : 1, slot[size_t(i)]);
        n_first = 1;
        if (i != early_seq[0]) n_first = 0;
      } else {
        n_first = pre;
      }
    } else if (ctx->pre_n > 0) {
      ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_precopy, 0), "wait");
    }
    ctx->pre_n = 0;
    if (reorder && early_seq.size() > 1) {
      // leaf closure of every contraction (memoised over nodes), restricted to early leaves
      std::vector<int32_t> early_of_node(g.nodes.size(), -1);
      for (size_t k = 0; k < early_seq.size(); ++k) early_of_node[size_t(ops[size_t(early_seq[k])].node)] = int32_t(k);
      std::vector<std::vector<int32_t>> leaves(g.nodes.size());
      std::vector<uint8_t> blocked(g.nodes.size(), 0);   // needs a leaf that is not early
      for (int32_t u : g.topo) {
        const Node& n = g.nodes[size_t(u)];
        if (n.leaf()) {
          if (early_of_node[size_t(u)] >= 0) leaves[size_t(u)] = {early_of_node[size_t(u)]};
          else blocked[size_t(u)] = 1;
          continue;
        }
        auto& v = leaves[size_t(u)];
        v = leaves[size_t(n.l)];
        v.insert(v.end(), leaves[size_t(n.r)].begin(), leaves[size_t(n.r)].end());
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        blocked[size_t(u)] = blocked[size_t(n.l)] | blocked[size_t(n.r)];
      }
      std::vector<int32_t> contr;
      std::vector<double> cost;
      for (int32_t i = 0; i < n_ops; ++i) {
        const PhysOp& op = ops[size_t(i)];
        if (op.kind != OP_CONTRACT || blocked[size_t(op.node)]) continue;
        const Node& n = g.nodes[size_t(op.node)];
        contr.push_back(op.node);
        cost.push_back(node_flops(n, g.Lt, g.N, g.S) / 37e12 + node_hbm_bytes(n, g.Lt, g.N, g.S) / 6.5e12);
      }
      const size_t ne = early_seq.size();
      std::vector<std::vector<int32_t>> users(ne);
      std::vector<int32_t> missing(contr.size());
      for (size_t c = 0; c < contr.size(); ++c) {
        missing[c] = int32_t(leaves[size_t(contr[c])].size());
        for (int32_t e : leaves[size_t(contr[c])]) users[size_t(e)].push_back(int32_t(c));
      }
      std::vector<double> score(ne, 0.0);
      for (size_t e = 0; e < ne; ++e)
        for (int32_t c : users[e])
          if (missing[size_t(c)] == 1) score[e] += cost[size_t(c)];
      std::vector<uint8_t> taken(ne, 0);
      std::vector<int32_t> out;
      for (size_t step = 0; step < ne; ++step) {
        size_t best = ne;
        if (step < size_t(n_first)) {
          best = step;                                // early_seq[step], already on its way
        } else {
          for (size_t e = 0; e < ne; ++e)
            if (!taken[e] && (best == ne || score[e] > score[best])) best = e;
        }
        taken[best] = 1;
        out.push_back(early_seq[best]);
        for (int32_t c : users[best]) {
          if (--missing[size_t(c)] == 1)
            for (int32_t e : leaves[size_t(contr[size_t(c)])])
              if (!taken[size_t(e)]) score[size_t(e)] += cost[size_t(c)];
        }
      }
      early_seq.swap(out);
    }
    // the last copies of the order gate the work left at the end: split them into time-slice
    // chunks (each a flag value; their consumers wait only for the chunk holding their slice)
    // so that work starts while the rest of the leaf is still in flight.  CC_H2D_TAIL copies
    // x CC_H2D_TAIL_CHUNKS chunks (every chunk costs one stream memory operation).
    const int tail = getenv("CC_H2D_TAIL") ? atoi(getenv("CC_H2D_TAIL")) : 0;
    const int tail_c = getenv("CC_H2D_TAIL_CHUNKS") ? atoi(getenv("CC_H2D_TAIL_CHUNKS")) : 4;
    for (int k = 0; k < tail && k < int(early_seq.size()) && tail_c > 1; ++k) {
      const int32_t i = early_seq[early_seq.size() - 1 - size_t(k)];
      const PhysOp& op = ops[size_t(i)];
      const int64_t C = std::min<int64_t>(Lt, tail_c);
      if (target[size_t(i)] == 1 && Lt > 1 && Lt % C == 0 && op.bytes % Lt == 0) target[size_t(i)] = -int32_t(C);
    }
  }
  // early copies: zero the sync area on the H2D stream, then start the early copies, each
  // followed by its flag write, so they overlap the rest of the host-side preparation; the
  // compute stream waits for the zeroing only.
  ctx->df_early.assign(size_t(n_ops), 0);
  ctx->df_early_active = false;
  if (early && !early_seq.empty()) {
    if (n_first == 0) {
      ck(cudaEventRecord(ctx->ev_pre, ctx->cs), "event");        // after all earlier work on cs
      ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_pre, 0), "wait");
      ck(cudaMemsetAsync(ctx->df_sync_base, 0, sz_sync, ctx->hs), "memset");
    }
    ck(cudaEventRecord(ctx->ev_pre, ctx->hs), "event");          // after the zeroing (and copy 0)
    ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_pre, 0), "wait");
    const bool dual = dual_h2d();
    if (dual) {
      ensure_hs2(ctx);
      ck(cudaStreamWaitEvent(ctx->hs2, ctx->ev_pre, 0), "wait");
    }
    size_t q = 0, q_issued = 0;
    for (int32_t i : early_seq) {
      const PhysOp& op = ops[size_t(i)];
      ctx->df_early[size_t(i)] = 1;
      if (q_issued++ < size_t(n_first)) continue;     // enqueued before the ordering
      const auto ep = copy_endpoints(ctx, op);
      enqueue_copy(ctx, (dual && (q++ & 1)) ? ctx->hs2 : ctx->hs, ep.first, ep.second, size_t(op.bytes),
                   cudaMemcpyHostToDevice, target[size_t(i)] < 0 ? -target[size_t(i)] : 1, slot[size_t(i)]);
    }
    if (dual) {                                   // rejoin: later hs work follows every early copy
      ck(cudaEventRecord(ctx->ev_hs2, ctx->hs2), "event");
      ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_hs2, 0), "wait");
    }
    ctx->df_early_active = true;
  }
  tmr.lap("early copies");
  // 1. data dependencies over the device pool and the host pool
  RWTracker dev(ctx->pool_bytes), host(std::max<int64_t>(ctx->pp.host_pool_bytes, 1));
  std::vector<std::vector<int32_t>> deps(static_cast<size_t>(n_ops));
  // writers of contraction operands: pool writer op, -1 never written, -2 caller device leaf
  std::vector<int32_t> wr_a(size_t(n_ops), -1), wr_b(size_t(n_ops), -1);
  for (int32_t i = 0; i < n_ops; ++i) {
    const PhysOp& op = ops[size_t(i)];
    const Node& n = g.nodes[size_t(op.node)];
    const int64_t rb = round_up(n.size, ALIGN);
    auto& d = deps[size_t(i)];
    if (op.kind == OP_H2D && op.stream != S_NONE) {
      dev.write(op.dev_off, rb, i, d);
      if (op.host_off >= 0) host.read(op.host_off, rb, i, d);
    } else if (op.kind == OP_D2H) {
      dev.read(op.dev_off, rb, i, d);
      host.write(op.host_off, rb, i, d);
    } else if (op.kind == OP_CONTRACT) {
      const int64_t sa = round_up(g.nodes[size_t(n.l)].size, ALIGN), sb = round_up(g.nodes[size_t(n.r)].size, ALIGN);
      wr_a[size_t(i)] = op.loc_a == LOC_POOL ? dev.last_writer(op.off_a, sa) : (op.loc_a == LOC_DEVLEAF ? -2 : -1);
      wr_b[size_t(i)] = op.loc_b == LOC_POOL ? dev.last_writer(op.off_b, sb) : (op.loc_b == LOC_DEVLEAF ? -2 : -1);
      if (op.loc_a == LOC_POOL) dev.read(op.off_a, sa, i, d);
      if (op.loc_b == LOC_POOL) dev.read(op.off_b, sb, i, d);
      if (op.dev_off >= 0) dev.write(op.dev_off, rb, i, d);
    }
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    d.erase(std::remove(d.begin(), d.end(), i), d.end());
  }
  // 1a. trace fusion.  A TR_MM op whose later operand is written by a GEMM op G (MM1 / BB2
  // output, full-K tiles) while its other operand was written before G (or is a caller device
  // leaf) is computed inside G's tiles: each output tile dots its registers with the matching
  // transposed tile of the other operand (tr(XY) = sum_ij X_ij Y_ji), so the trace never
  // reads G's output back from HBM and needs no work items of its own.  Its data dependencies
  // move to G (G now also waits for the other operand's writer, which precedes G in plan
  // order), and everything that waited for the TR op waits for G instead.  CC_DF_FUSE_TR=0
  // turns it off.
  std::vector<int32_t> fuse_host(size_t(n_ops), -1);
  std::vector<std::vector<int32_t>> fused_of(static_cast<size_t>(n_ops));
  {
    constexpr size_t MAX_FUSED = 16;
    // default off: on c2 the fused partner stages come in bursts the 6-stage ring cannot hide
    // (4.89 ms vs 4.64 ms unfused, profiles/r01 notes); kept for larger N and as an option
    const bool fuse = getenv("CC_DF_FUSE_TR") ? atoi(getenv("CC_DF_FUSE_TR")) != 0 : false;
    for (int32_t i = 0; fuse && i < n_ops; ++i) {
      const PhysOp& op = ops[size_t(i)];
      if (op.kind != OP_CONTRACT || g.nodes[size_t(op.node)].op != CC_TR_MM) continue;
      const Node& n = g.nodes[size_t(op.node)];
      const int32_t wa = wr_a[size_t(i)], wb = wr_b[size_t(i)];
      int32_t G, other, gnode;
      if (wa >= 0 && wa > wb) {
        G = wa; other = wb; gnode = n.l;
      } else if (wb >= 0 && wb > wa) {
        G = wb; other = wa; gnode = n.r;
      } else {
        continue;
      }
      if (other == -1) continue;   // other operand never written in the pool (not resident)
      const PhysOp& og = ops[size_t(G)];
      if (og.kind != OP_CONTRACT || og.node != gnode) continue;
      const int gop = g.nodes[size_t(gnode)].op;
      if (gop != CC_MM1 && gop != CC_BB2) continue;
      int64_t tiles, KT, chunks;
      df_gemm_geometry(problem_for(gop, Lt, N, g.S, nullptr, nullptr, nullptr), tiles, KT, chunks, ctx->num_sms);
      if (chunks != 1 || fused_of[size_t(G)].size() >= MAX_FUSED) continue;
      fuse_host[size_t(i)] = G;
      fused_of[size_t(G)].push_back(i);
      if (other >= 0) {
        auto& dg = deps[size_t(G)];
        if (std::find(dg.begin(), dg.end(), other) == dg.end()) dg.push_back(other);
      }
    }
  }
  tmr.lap("rw deps");
  // 1b. copy issue order per stream: the early H2D copies (chosen and possibly already
  // enqueued in step 0) first, in their order, then the other copies in plan order.
  std::vector<int32_t> copy_seq[3];
  std::vector<int64_t> copy_pos(size_t(n_ops), 0);   // H2D issue position (0 for non-copies)
  {
    copy_seq[S_H2D] = early_seq;
    for (int32_t i = 0; i < n_ops; ++i) {
      const int st = ops[size_t(i)].stream;
      if ((st == S_H2D && !is_early[size_t(i)]) || st == S_D2H) copy_seq[st].push_back(i);
    }
    const auto& h = copy_seq[S_H2D];
    for (size_t k = 0; k < h.size(); ++k) copy_pos[size_t(h[k])] = int64_t(k) + 1;
  }
  // 2. work items
  std::vector<DfOp> gops, tops;
  std::vector<int32_t> gplan, tplan;   // plan op index of each DfOp (queue order)
  std::vector<uint8_t> tmaps;
  int64_t g_items = 0, t_items = 0;
  int64_t n_chunked = 0, n_traced = 0;
  std::vector<int32_t> chunk_ring_user(size_t(DF_CHUNK_RING), -1), trace_ring_user(size_t(DF_TRACE_RING), -1);
  std::vector<std::vector<int32_t>> ring_deps(static_cast<size_t>(n_ops));
  std::vector<DfFused> fusedv;
  int64_t fused_part_bytes = 0;
  constexpr int64_t GC_WARPS = 8;   // consumer warps of the worker (per-warp fused partials)
  int BM, BN, BK, slot_doubles;
  df_gemm_tile_dims(&BM, &BN, &BK, &slot_doubles);
  for (int32_t i = 0; i < n_ops; ++i) {
    const PhysOp& op = ops[size_t(i)];
    if (op.stream == S_NONE || op.kind != OP_CONTRACT) continue;
    const Node& n = g.nodes[size_t(op.node)];
    const void* a = op.loc_a == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.l)] : ctx->arena + op.off_a;
    const void* b = op.loc_b == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.r)] : ctx->arena + op.off_b;
    if (fuse_host[size_t(i)] >= 0) continue;   // fused TR: computed by its host GEMM's tiles
    DfOp d{};
    d.sync_id = slot[size_t(i)];
    d.slice_sync = -1;
    if (n.op == CC_TR_MM) {
      const int64_t P = df_trace_pieces(Lt, N);
      d.kind = 1;
      d.n_items = int32_t(Lt * P);
      d.first_item = g_items;
      d.A = a;
      d.B = b;
      d.out = ctx->roots + int64_t(g.tree_of_root[size_t(op.node)]) * Lt;
      d.N = N;
      d.Lt = Lt;
      d.nb = int32_t((N + 31) / 32);
      d.P = int32_t(P);
      // partial slots (P > 1) come from a ring assigned in queue order below
      d.tmap = int32_t(tmaps.size() / 256);
      tmaps.resize(tmaps.size() + 256);
      if (!df_encode_trace_maps(tmaps.data() + size_t(d.tmap) * 256, a, b, Lt, N))
        throw Error(CC_E_CUDA, "TMA descriptor encoding failed");
      g_items += d.n_items;
      df_index[size_t(i)] = int32_t(gops.size());
      gops.push_back(d);
      gplan.push_back(i);
    } else {
      void* out = ctx->arena + op.dev_off;
      ZgemmProblem p = problem_for(n.op, Lt, N, g.S, a, b, out);
      int64_t tiles, KT, chunks;
      df_gemm_geometry(p, tiles, KT, chunks, ctx->num_sms);
      d.kind = 0;
      d.n_items = int32_t(tiles * chunks);
      if (slice_slot[size_t(i)] >= 0 && p.batch == Lt && d.n_items % Lt == 0) {
        d.slice_sync = slice_slot[size_t(i)];
        items_per_slice[size_t(i)] = int32_t(d.n_items / Lt);
      }
      d.first_item = g_items;
      d.tiles_m = int32_t((p.M + BM - 1) / BM);
      d.tiles_n = int32_t((p.Nn + BN - 1) / BN);
      d.kt_per_o = int32_t((p.Kin + BK - 1) / BK);
      d.KT = int32_t(KT);
      d.n_chunks = int32_t(chunks);
      d.M = p.M;
      d.Nn = p.Nn;
      d.ldc = p.ldc;
      d.sCb = p.sCb;
      d.C = out;
      // chunk-partial slots (chunks > 1) come from a ring assigned in queue order below
      d.tmap = int32_t(tmaps.size() / 256);
      tmaps.resize(tmaps.size() + 256);
      if (!df_encode_maps(tmaps.data() + size_t(d.tmap) * 256, p.A, p.B, p.M, p.Nn, p.Kin, p.Ko, p.batch, p.lda,
                          p.sAo, p.sAb, p.ldb, p.sBo, p.sBb))
        throw Error(CC_E_CUDA, "TMA descriptor encoding failed");
      if (!fused_of[size_t(i)].empty()) {
        d.fuse_begin = int32_t(fusedv.size());
        d.fuse_count = int32_t(fused_of[size_t(i)].size());
        for (int32_t f : fused_of[size_t(i)]) {
          const PhysOp& of = ops[size_t(f)];
          const Node& nf = g.nodes[size_t(of.node)];
          const bool g_left = nf.l == op.node;     // G's output is the TR's left operand
          const void* x = g_left ? (of.loc_b == LOC_DEVLEAF ? ctx->leaf_dev[size_t(nf.r)] : ctx->arena + of.off_b)
                                 : (of.loc_a == LOC_DEVLEAF ? ctx->leaf_dev[size_t(nf.l)] : ctx->arena + of.off_a);
          DfFused fz{};
          fz.tmap = int32_t(tmaps.size() / 256);
          tmaps.resize(tmaps.size() + 256);
          if (!df_encode_partner_map(tmaps.data() + size_t(fz.tmap) * 256, x, Lt, N))
            throw Error(CC_E_CUDA, "TMA descriptor encoding failed");
          fz.tiles = d.tiles_m * d.tiles_n;
          fz.part = reinterpret_cast<double2*>(fused_part_bytes);   // offset; patched at upload
          fused_part_bytes += Lt * fz.tiles * GC_WARPS * 16;
          fz.root = ctx->roots + int64_t(g.tree_of_root[size_t(of.node)]) * Lt;
          fusedv.push_back(fz);
        }
      }
      g_items += d.n_items;
      df_index[size_t(i)] = int32_t(gops.size());
      gops.push_back(d);
      gplan.push_back(i);
    }
    target[size_t(i)] = d.n_items;
  }
  // fused TR ops alias their host GEMM's completion (dependents wait for the GEMM)
  for (int32_t i = 0; i < n_ops; ++i)
    if (fuse_host[size_t(i)] >= 0) {
      slot[size_t(i)] = slot[size_t(fuse_host[size_t(i)])];
      target[size_t(i)] = target[size_t(fuse_host[size_t(i)])];
    }
  tmr.lap("items+tmaps");
  std::vector<int64_t> qpos(size_t(n_ops), INT64_MAX);   // merged queue position of compute ops
  // 3. queue order: a topological order of the plan's ops (compute and copy; consecutive
  // copies on one stream are chained, since a copy stream runs in plan order) that delays each
  // TR_MM op by DF_TR_DELAY compute positions, so a trace item is usually claimed after its
  // operand GEMMs completed (no worker blocks on it) while the GEMMs behind it keep the DMMA
  // pipes busy.  Any topological order keeps the dataflow deadlock-free (dataflow.hpp).
  {
    static const int64_t delay = getenv("CC_DF_TR_DELAY") ? atoll(getenv("CC_DF_TR_DELAY")) : 8;
    std::vector<std::vector<int32_t>> succ(static_cast<size_t>(n_ops));
    std::vector<int32_t> indeg(static_cast<size_t>(n_ops), 0), rank(static_cast<size_t>(n_ops), 0);
    std::vector<int32_t> chain_prev(size_t(n_ops), -1);   // previous copy on the same stream (issue order)
    for (int st : {int(S_H2D), int(S_D2H)})
      for (size_t k = 1; k < copy_seq[st].size(); ++k) chain_prev[size_t(copy_seq[st][k])] = copy_seq[st][k - 1];
    // avail: the H2D issue position after which an op's inputs can all be there
    std::vector<int64_t> avail(size_t(n_ops), 0);
    int32_t r = 0;
    for (int32_t i = 0; i < n_ops; ++i) {
      if (slot[size_t(i)] < 0) continue;
      rank[size_t(i)] = r;
      if (ops[size_t(i)].kind == OP_CONTRACT) ++r;
      std::vector<int32_t> pre = deps[size_t(i)];
      pre.insert(pre.end(), ring_deps[size_t(i)].begin(), ring_deps[size_t(i)].end());
      if (ops[size_t(i)].kind != OP_CONTRACT && chain_prev[size_t(i)] >= 0) pre.push_back(chain_prev[size_t(i)]);
      for (int32_t j : pre) avail[size_t(i)] = std::max(avail[size_t(i)], std::max(avail[size_t(j)], copy_pos[size_t(j)]));
      std::sort(pre.begin(), pre.end());
      pre.erase(std::unique(pre.begin(), pre.end()), pre.end());
      for (int32_t j : pre)
        if (slot[size_t(j)] >= 0) {
          succ[size_t(j)].push_back(i);
          ++indeg[size_t(i)];
        }
    }
    // priority: inputs' availability first (copy issue order), then plan rank (+ the TR delay)
    auto key = [&](int32_t i) {
      const PhysOp& op = ops[size_t(i)];
      const bool tr = op.kind == OP_CONTRACT && g.nodes[size_t(op.node)].op == CC_TR_MM;
      return avail[size_t(i)] * (int64_t(n_ops) + delay + 1) + int64_t(rank[size_t(i)]) + (tr ? delay : 0);
    };
    std::priority_queue<std::pair<int64_t, int32_t>, std::vector<std::pair<int64_t, int32_t>>, std::greater<>> ready;
    for (int32_t i = 0; i < n_ops; ++i)
      if (slot[size_t(i)] >= 0 && indeg[size_t(i)] == 0) ready.push({key(i), i});
    std::vector<int32_t> order;
    while (!ready.empty()) {
      const int32_t i = ready.top().second;
      ready.pop();
      if (ops[size_t(i)].kind == OP_CONTRACT) {
        qpos[size_t(i)] = int64_t(order.size());
        order.push_back(i);
      }
      for (int32_t k : succ[size_t(i)])
        if (--indeg[size_t(k)] == 0) ready.push({key(k), k});
    }
    size_t n_fused_ops = 0;
    for (int32_t i = 0; i < n_ops; ++i) n_fused_ops += fuse_host[size_t(i)] >= 0;
    if (order.size() != gops.size() + n_fused_ops) throw Error(CC_E_STATE, "dataflow: dependency cycle");
    std::vector<DfOp> nops, tops_v;
    std::vector<int32_t> nplan, tplan_v;
    int64_t first = 0, tfirst = 0;
    for (int32_t i : order) {
      if (df_index[size_t(i)] < 0) continue;   // fused TR (no items)
      DfOp d = gops[size_t(df_index[size_t(i)])];
      if (d.kind == 0) {
        d.first_item = first;
        first += d.n_items;
        nops.push_back(d);
        nplan.push_back(i);
      } else {
        d.first_item = tfirst;
        tfirst += d.n_items;
        tops_v.push_back(d);
        tplan_v.push_back(i);
      }
    }
    gops.swap(nops);
    gplan.swap(nplan);
    tops.swap(tops_v);
    tplan.swap(tplan_v);
    g_items = first;
    t_items = tfirst;
    // Workspace rings (chunk partials of k-split GEMM ops, slice partials of TR ops split in
    // P > 1 pieces), assigned in queue order: the op taking a slot depends on the slot's
    // previous user, which is earlier in the same queue — the queue order stays topological.
    for (size_t k = 0; k < gops.size(); ++k) {
      if (gops[k].n_chunks <= 1) continue;
      const int64_t r = n_chunked++ % DF_CHUNK_RING;
      char* base = ctx->df_chunk_ws + r * (ctx->df_chunk_slot + ctx->df_chunk_cnt_slot);
      gops[k].part = base;
      gops[k].tile_cnt = reinterpret_cast<int*>(base + ctx->df_chunk_slot);
      if (chunk_ring_user[size_t(r)] >= 0) ring_deps[size_t(gplan[k])].push_back(chunk_ring_user[size_t(r)]);
      chunk_ring_user[size_t(r)] = gplan[k];
    }
    for (size_t k = 0; k < tops.size(); ++k) {
      if (tops[k].P <= 1) continue;
      const int64_t r = n_traced++ % DF_TRACE_RING;
      char* base = ctx->df_trace_ws + r * ctx->df_trace_slot;
      tops[k].tr_cnt = reinterpret_cast<int*>(base);
      tops[k].tr_part = base + round_up(Lt * 4, ALIGN);
      if (trace_ring_user[size_t(r)] >= 0) ring_deps[size_t(tplan[k])].push_back(trace_ring_user[size_t(r)]);
      trace_ring_user[size_t(r)] = tplan[k];
    }
  }
  tmr.lap("queue order");
  // 4. dependency lists of compute ops, wait lists of copies
  std::vector<int32_t> dep_slot, dep_target;
  auto fill_deps = [&](std::vector<DfOp>& v, const std::vector<int32_t>& plan, bool traces) {
    for (size_t k = 0; k < v.size(); ++k) {
      const int32_t i = plan[k];
      v[k].dep_begin = int32_t(dep_slot.size());
      std::vector<int32_t> all = deps[size_t(i)];
      all.insert(all.end(), ring_deps[size_t(i)].begin(), ring_deps[size_t(i)].end());
      std::sort(all.begin(), all.end());
      all.erase(std::unique(all.begin(), all.end()), all.end());
      for (int32_t j : all) {
        if (slot[size_t(j)] < 0) continue;
        if (traces && items_per_slice[size_t(j)] > 0) {   // a trace reads slice t of this GEMM's output
          dep_slot.push_back(slice_slot[size_t(j)]);
          dep_target.push_back(-(1 << 20) - items_per_slice[size_t(j)]);
          continue;
        }
        dep_slot.push_back(slot[size_t(j)]);
        dep_target.push_back(target[size_t(j)]);
      }
      v[k].dep_count = int32_t(dep_slot.size()) - v[k].dep_begin;
    }
  };
  fill_deps(gops, gplan, false);
  fill_deps(tops, tplan, true);
  ctx->df_copies.clear();
  std::vector<int32_t> copy_index(static_cast<size_t>(n_ops), -1);
  for (int32_t i = 0; i < n_ops; ++i) {
    const PhysOp& op = ops[size_t(i)];
    if (op.stream != S_H2D && op.stream != S_D2H) continue;
    const Node& n = g.nodes[size_t(op.node)];
    cc_ctx::DfCopy c;
    c.op = i;
    c.stream = op.stream;
    c.bytes = size_t(op.bytes);
    c.flag_slot = slot[size_t(i)];
    {
      const auto ep = copy_endpoints(ctx, op);
      c.src = ep.first;
      c.dst = ep.second;
    }
    for (int32_t j : deps[size_t(i)]) {
      const PhysOp& oj = ops[size_t(j)];
      if (oj.kind == OP_CONTRACT) {
        c.wait_values.push_back({slot[size_t(j)], target[size_t(j)]});
      } else if (oj.stream != op.stream && copy_index[size_t(j)] >= 0) {
        c.wait_events.push_back(copy_index[size_t(j)]);
        ctx->df_copies[size_t(copy_index[size_t(j)])].source = true;
      }
    }
    if (target[size_t(i)] < 0) c.chunks = -target[size_t(i)];
    copy_index[size_t(i)] = int32_t(ctx->df_copies.size());
    ctx->df_copies.push_back(std::move(c));
  }
  {
    const size_t nc = ctx->df_copies.size();
    std::vector<int32_t> seq[3];
    for (int st : {int(S_H2D), int(S_D2H)})
      for (int32_t i : copy_seq[st]) seq[st].push_back(copy_index[size_t(i)]);
    // merge the two streams' sequences so every event source is enqueued before its waiters
    std::vector<uint8_t> done(nc, 0);
    size_t p[3] = {0, 0, 0};
    ctx->df_issue.clear();
    while (ctx->df_issue.size() < nc) {
      int pick = -1;
      for (int st : {int(S_H2D), int(S_D2H)}) {
        if (p[st] >= seq[st].size()) continue;
        const auto& c = ctx->df_copies[size_t(seq[st][p[st]])];
        bool ok = true;
        for (int32_t e : c.wait_events) ok = ok && done[size_t(e)];
        if (ok && (pick < 0 || seq[st][p[st]] < seq[pick][p[pick]])) pick = st;
      }
      if (pick < 0) throw Error(CC_E_STATE, "dataflow: copy order cycle");
      const int32_t k = seq[pick][p[pick]++];
      done[size_t(k)] = 1;
      ctx->df_issue.push_back(k);
    }
  }
  if (!ctx->df_copies.empty() && (!df_wait_fn() || !df_write_fn()))
    throw Error(CC_E_CUDA, "stream memory operations (cuStreamWaitValue32) unavailable");
  ctx->df_events.assign(ctx->df_copies.size(), nullptr);
  for (size_t k = 0; k < ctx->df_copies.size(); ++k)
    if (ctx->df_copies[k].source) ck(cudaEventCreateWithFlags(&ctx->df_events[k], cudaEventDisableTiming), "event");
  tmr.lap("deps+copies+events");
  // 5. upload metadata: [heads | sync][gops][tops][dep_slot][dep_target][tmaps]
  const size_t sz_g = round_up(int64_t(std::max<size_t>(gops.size(), 1) * sizeof(DfOp)), 256);
  const size_t sz_t = round_up(int64_t(std::max<size_t>(tops.size(), 1) * sizeof(DfOp)), 256);
  const size_t sz_d = round_up(int64_t(std::max<size_t>(dep_slot.size(), 1) * 4), 256);
  const size_t sz_m = round_up(int64_t(std::max<size_t>(tmaps.size(), 256)), 256);
  std::vector<int32_t> gitem_op(size_t(std::max<int64_t>(g_items, 1)), 0), titem_op(size_t(std::max<int64_t>(t_items, 1)), 0);
  for (size_t k = 0; k < gops.size(); ++k)
    std::fill(gitem_op.begin() + gops[k].first_item, gitem_op.begin() + gops[k].first_item + gops[k].n_items, int32_t(k));
  for (size_t k = 0; k < tops.size(); ++k)
    std::fill(titem_op.begin() + tops[k].first_item, titem_op.begin() + tops[k].first_item + tops[k].n_items, int32_t(k));
  const size_t sz_gi = round_up(int64_t(gitem_op.size() * 4), 256), sz_ti = round_up(int64_t(titem_op.size() * 4), 256);
  const size_t sz_f = round_up(int64_t(std::max<size_t>(fusedv.size(), 1) * sizeof(DfFused)), 256);
  const size_t total = sz_g + sz_t + 2 * sz_d + sz_m + sz_gi + sz_ti + sz_f;
  // device region: the top of the pool when the plan's high water leaves room (no allocation
  // on the execute path), else a cudaMalloc
  const int64_t meta_off = (int64_t(ctx->df_sync_base - ctx->arena) - int64_t(total)) / 256 * 256;
  if (meta_off >= ctx->pp.pool_high_water) {
    ctx->df_meta = ctx->arena + meta_off;
    ctx->df_meta_owned = false;
  } else {
    ck(cudaMalloc(reinterpret_cast<void**>(&ctx->df_meta), total), "dataflow metadata");
    ctx->df_meta_owned = true;
  }
  ctx->df_meta_bytes = total;
  // fused-trace partials ([Lt][tiles][warps] per fused TR, written before read: no upload)
  if (ctx->df_fpart && ctx->df_fpart_owned) cudaFree(ctx->df_fpart);
  ctx->df_fpart = nullptr;
  ctx->df_fpart_owned = false;
  if (fused_part_bytes > 0) {
    const int64_t fp_off = (meta_off - fused_part_bytes) / 256 * 256;
    if (!ctx->df_meta_owned && fp_off >= ctx->pp.pool_high_water) {
      ctx->df_fpart = ctx->arena + fp_off;
    } else {
      ck(cudaMalloc(reinterpret_cast<void**>(&ctx->df_fpart), size_t(fused_part_bytes)), "fused trace partials");
      ctx->df_fpart_owned = true;
    }
    for (auto& fz : fusedv) fz.part = reinterpret_cast<double2*>(ctx->df_fpart + reinterpret_cast<intptr_t>(fz.part));
  }
  char* m = ctx->df_meta;
  unsigned long long* heads = reinterpret_cast<unsigned long long*>(ctx->df_sync_base);
  char* pg = m;
  char* pt = pg + sz_g;
  char* pds = pt + sz_t;
  char* pdt = pds + sz_d;
  char* pm = pdt + sz_d;
  char* pgi = pm + sz_m;
  char* pti = pgi + sz_gi;
  char* pf = pti + sz_ti;
  {
    // one host image, one copy, ordered on the compute stream before the worker launch
    if (ctx->df_meta_img_bytes < total) {
      if (ctx->df_meta_img) cudaFreeHost(ctx->df_meta_img);
      ctx->df_meta_img = nullptr;
      ctx->df_meta_img_bytes = 0;
      ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->df_meta_img), total, cudaHostAllocDefault), "metadata staging");
      ctx->df_meta_img_bytes = total;
    } else {
      ck(cudaEventSynchronize(ctx->ev_meta), "metadata staging");   // the previous upload has read it
    }
    struct Img {
      char* p;
      char* data() { return p; }
    } img{ctx->df_meta_img};
    std::memset(img.data(), 0, total);
    auto put = [&](char* dst, const void* src, size_t n) {
      if (n) std::memcpy(img.data() + (dst - m), src, n);
    };
    put(pgi, gitem_op.data(), gitem_op.size() * 4);
    put(pti, titem_op.data(), titem_op.size() * 4);
    put(pg, gops.data(), gops.size() * sizeof(DfOp));
    put(pt, tops.data(), tops.size() * sizeof(DfOp));
    put(pds, dep_slot.data(), dep_slot.size() * 4);
    put(pdt, dep_target.data(), dep_target.size() * 4);
    put(pm, tmaps.data(), tmaps.size());
    put(pf, fusedv.data(), fusedv.size() * sizeof(DfFused));
    // SM-driven upload on the compute stream: the copy engines may be busy with early leaf copies
    ck(launch_upload(m, img.data(), total, ctx->num_sms, ctx->cs), "dataflow metadata upload");
    ck(cudaEventRecord(ctx->ev_meta, ctx->cs), "event");
  }
  DfArgs& da = ctx->df_gemm;
  da.dep_slot = reinterpret_cast<const int32_t*>(pds);
  da.dep_target = reinterpret_cast<const int32_t*>(pdt);
  da.tmaps = pm;
  da.sync = ctx->df_sync;
  da.fused = reinterpret_cast<const DfFused*>(pf);
  ctx->df_n_fused = int32_t(fusedv.size());
  da.q = DfQueue{reinterpret_cast<const DfOp*>(pg), reinterpret_cast<const int32_t*>(pgi), int32_t(gops.size()),
                 g_items, heads};
  da.qt = DfQueue{reinterpret_cast<const DfOp*>(pt), reinterpret_cast<const int32_t*>(pti), int32_t(tops.size()),
                  t_items, heads + 1};
  {
    auto env_int = [](const char* k, int dflt, int lo, int hi) {
      const char* v = getenv(k);
      return std::min(std::max(v ? atoi(v) : dflt, lo), hi);
    };
    // TR_MM stages the issuer may put between GEMM k-tiles (fixed point, 1/8): by default
    // 1.12 x the plan's trace-stage / k-tile-stage ratio, so the traces keep pace with the
    // GEMMs (c2: 1.56 -> 1.75; measured on c2: 1.5 / 1.75 / 2 / 2.5 -> 4.45 / 4.38 / 4.43 /
    // 4.62 ms); CC_DF_TR_RATIO overrides
    double g_st = 0, t_st = 0;
    for (const auto& o : gops) g_st += double(o.n_items / std::max(o.n_chunks, 1)) * o.KT;
    for (const auto& o : tops) t_st += double(o.Lt) * o.nb * o.nb;
    const double auto_ratio = g_st > 0 && t_st > 0 ? std::min(std::max(1.12 * t_st / g_st, 0.25), 8.0) : 2.0;
    const char* rv = getenv("CC_DF_TR_RATIO");
    da.tr_ratio8 = std::min(std::max(int(std::lround((rv ? atof(rv) : auto_ratio) * 8.0)), 0), 512);
    da.Lt = int32_t(Lt);
    da.ahead_g = env_int("CC_DF_AHEAD_G", 2, 1, 4);
    da.ahead_t = env_int("CC_DF_AHEAD_T", 2, 1, 4);
  }
  ctx->df_gemm_items = g_items;
  ctx->df_trace_items = t_items;
  da.prof = nullptr;
  da.prof_t = nullptr;
  if (!ctx->cs2) {
    ck(cudaStreamCreateWithFlags(&ctx->cs2, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ctx->ev_cs2, cudaEventDisableTiming), "event");
  }
  tmr.lap("upload");
  ctx->df_valid = true;
}

// Enqueues one dataflow replay; returns the number of kernel launches.
int issue_dataflow(cc_ctx* ctx, bool time_copies = false) {
  const Dag& g = *ctx->dag;
  int nl = 0;
  static const bool dbg = getenv("CC_DEBUG") != nullptr;
#define DBG(...) do { if (dbg) { fprintf(stderr, "[cc] " __VA_ARGS__); fputc('\n', stderr); fflush(stderr); } } while (0)
  PhaseTimer tmr("issue_dataflow");
  DBG("issue_dataflow: %zu copies, %lld gemm items, %lld trace items", ctx->df_copies.size(),
      (long long)ctx->df_gemm_items, (long long)ctx->df_trace_items);
  if (!ctx->df_early_active) ck(cudaMemsetAsync(ctx->df_sync_base, 0, ctx->df_sync_bytes, ctx->cs), "memset");
  ck(cudaEventRecord(ctx->ev_start, ctx->cs), "event");
  ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_start, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->ds, ctx->ev_start, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->cs2, ctx->ev_start, 0), "wait");
  // The worker goes first: copy streams may block on stream memory ops waiting for its
  // counters, and a driver can stall the host's enqueue of further memory ops until the
  // device makes progress — so the kernel they wait for must already be queued.
  if (ctx->df_gemm_items + ctx->df_trace_items > 0) {
    ck(df_launch(ctx->df_gemm, ctx->num_sms, ctx->cs), "dataflow worker");
    DBG("worker launched");
    ++nl;
    if (ctx->df_n_fused > 0) {
      ck(df_launch_fused_finish(ctx->df_gemm.fused, ctx->df_n_fused, g.Lt, ctx->cs), "fused trace finish");
      ++nl;
    }
  }
  cudaStream_t st[3] = {ctx->cs, ctx->hs, ctx->ds};
  const bool dual = dual_h2d();
  if (dual) {
    ensure_hs2(ctx);
    ck(cudaStreamWaitEvent(ctx->hs2, ctx->ev_start, 0), "wait");
  }
  size_t q = 0;
  for (const int32_t kk : ctx->df_issue) {
    const size_t k = size_t(kk);
    const auto& c = ctx->df_copies[k];
    cudaStream_t s = st[c.stream];
    // wait-free H2D copies (no event / value waits) alternate with the second H2D stream; any
    // copy that waits stays on hs, whose order the explicit waits already cover
    if (dual && c.stream == S_H2D && c.wait_events.empty() && c.wait_values.empty() && (q++ & 1)) s = ctx->hs2;
    for (int32_t e : c.wait_events) ck(cudaStreamWaitEvent(s, ctx->df_events[size_t(e)], 0), "wait");
    for (const auto& wv : c.wait_values)
      if (df_wait_fn()(s, reinterpret_cast<CUdeviceptr>(ctx->df_sync + wv.first), cuuint32_t(wv.second),
                       CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        throw Error(CC_E_CUDA, "cuStreamWaitValue32 failed");
    DBG("copy %zu: stream %d bytes %zu waits %zu/%zu", k, c.stream, c.bytes, c.wait_values.size(), c.wait_events.size());
    // copies started during preparation (flags included) are skipped
    if (!(ctx->df_early_active && ctx->df_early[size_t(c.op)]))
      enqueue_copy(ctx, s, c.src, c.dst, c.bytes, c.stream == S_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                   c.chunks, c.flag_slot);
    DBG("copy %zu enqueued", k);
    if (c.source) ck(cudaEventRecord(ctx->df_events[k], s), "event");
  }
  DBG("copies enqueued");
  if (dual) {
    ck(cudaEventRecord(ctx->ev_hs2, ctx->hs2), "event");
    ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_hs2, 0), "wait");
  }
  ctx->df_early_active = false;   // later replays copy everything and zero the sync area on cs
  if (time_copies) {
    ck(cudaEventRecord(ctx->ev_copy_h, ctx->hs), "event");
    ck(cudaEventRecord(ctx->ev_copy_d, ctx->ds), "event");
  }
  ctx->copy_timed = time_copies;
  tmr.lap("copies");
  DBG("workers launched");
  tmr.lap("worker");
  ck(cudaEventRecord(ctx->ev_cs2, ctx->cs2), "event");
  ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_cs2, 0), "wait");
  ck(launch_correlate(ctx->roots, ctx->corr, int64_t(g.corr_ids.size()), g.Lt, ctx->term_start, ctx->term_tree,
                      ctx->term_coef, ctx->cs),
     "correlate kernel");
  ++nl;
  ck(cudaEventRecord(ctx->ev_h_end, ctx->hs), "event");
  ck(cudaEventRecord(ctx->ev_d_end, ctx->ds), "event");
  ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_h_end, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_d_end, 0), "wait");
  return nl;
}

// Resets the Ozaki leaf-form cache for one execute (or one kernel-only capture): the free
// pool range above the plan's high water, below any dataflow metadata / sync area placed at
// the top of the pool.  CC_OZAKI_LEAF_CACHE=0 disables it.
void oz_cache_reset(cc_ctx* ctx) {
  const size_t n = ctx->dag->nodes.size();
  for (int k = 0; k < 6; ++k) {
    ctx->oz.form[k].assign(n, OzakiForm{nullptr, nullptr});
    ctx->oz.have[k].assign(n, 0);
  }
  int64_t end = ctx->pool_bytes;
  if (ctx->df_sync_base) end = std::min<int64_t>(end, ctx->df_sync_base - ctx->arena);
  if (ctx->df_meta && !ctx->df_meta_owned) end = std::min<int64_t>(end, ctx->df_meta - ctx->arena);
  if (ctx->df_fpart && !ctx->df_fpart_owned) end = std::min<int64_t>(end, reinterpret_cast<char*>(ctx->df_fpart) - ctx->arena);
  const char* env = getenv("CC_OZAKI_LEAF_CACHE");
  const bool off = env && atoi(env) == 0;
  if (ctx->oz_scratch_bytes > 0) {            // offsets relative to the arena base
    ctx->oz.off = ctx->oz_scratch - ctx->arena;
    ctx->oz.end = off ? ctx->oz.off : ctx->oz.off + ctx->oz_scratch_bytes;
  } else {
    ctx->oz.off = round_up(ctx->pp.pool_high_water, ALIGN);
    ctx->oz.end = off ? ctx->oz.off : end;
  }
}

// The A-form (as_b false) or B-form of operand node `u` of problem q (op kind `op`) if it is a
// leaf with room in the cache (made now, on the compute stream, at its first use), else nullptr.
const OzakiForm* oz_leaf_form(cc_ctx* ctx, int op, const ZgemmProblem& q, int32_t u, bool as_b) {
  const Dag& g = *ctx->dag;
  if (u < 0 || !g.nodes[size_t(u)].leaf()) return nullptr;
  const int k = 2 * oz_kind(op) + (as_b ? 1 : 0);
  if (ctx->oz.have[k][size_t(u)]) return &ctx->oz.form[k][size_t(u)];
  const int64_t bytes = round_up(int64_t(ozaki_form_bytes(q, OZAKI_SLICES, as_b)), ALIGN);
  if (ctx->oz.off + bytes > ctx->oz.end) return nullptr;
  ck(launch_ozaki_form(q, OZAKI_SLICES, as_b, ctx->arena + ctx->oz.off, &ctx->oz.form[k][size_t(u)], ctx->cs),
     "Ozaki leaf split");
  ctx->oz.off += bytes;
  ctx->oz.have[k][size_t(u)] = 1;
  return &ctx->oz.form[k][size_t(u)];
}

void launch_contract(cc_ctx* ctx, const Node& n, const void* a, const void* b, void* out, int64_t root_slot,
                     int* nl) {
  const Dag& g = *ctx->dag;
  if (n.op == CC_TR_MM) {
    ck(launch_trace(a, b, ctx->roots + root_slot * g.Lt, g.Lt, g.N, ctx->trace_ws, ctx->cs), "TR_MM kernel");
    ++*nl;
    return;
  }
  if (ctx->mm1_ozaki) {
    const ZgemmProblem q = problem_for(n.op, g.Lt, g.N, g.S, a, b, out);
    // forms only when the whole batch fits the workspace (else the engine splits per batch)
    const bool whole = ozaki_workspace_bytes(q, OZAKI_SLICES, g.Lt) <= ctx->gemm_ws_bytes;
    const OzakiForm* fa = whole ? oz_leaf_form(ctx, n.op, q, n.l, false) : nullptr;
    const OzakiForm* fb = whole ? oz_leaf_form(ctx, n.op, q, n.r, true) : nullptr;
    ck(launch_ozaki_gemm(q, OZAKI_SLICES, ctx->gemm_ws, ctx->gemm_ws_bytes, ctx->cs, fa, fb), "Ozaki GEMM");
    *nl += 6;   // (memset + colmax + 2 splits, or cached leaf forms made once) + GEMM (+ split-K reduce)
    return;
  }
  ZgemmProblem p = problem_for(n.op, g.Lt, g.N, g.S, a, b, out);
  ck(launch_zgemm(p, ctx->gemm_ws, ctx->gemm_ws_bytes, ctx->num_sms, ctx->cs, nl), "contraction kernel");
}

// Issues the plan on the three streams.  Returns the number of kernel launches.
int issue(cc_ctx* ctx, bool time_kernels, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* kev,
          std::vector<int>* kev_kind) {
  const Dag& g = *ctx->dag;
  const int64_t per_t_m = 16LL * g.N * g.N;
  cudaStream_t st[3] = {ctx->cs, ctx->hs, ctx->ds};
  int nl = 0;
  // CC_OPBYOP_H2D_STREAMS (1..4, default 1; c4 measured no gain: its copies wait for freed pool
  // memory, not behind each other): H2D copies round-robin over that many streams, with
  // their same-stream dependencies made explicit (op.same_deps), so a copy that waits for
  // memory to be freed does not hold back later copies that could already run
  static const int n_h2d = std::max(1, std::min(4, getenv("CC_OPBYOP_H2D_STREAMS") ? atoi(getenv("CC_OPBYOP_H2D_STREAMS")) : 1));
  cudaStream_t h2d[4] = {ctx->hs, nullptr, nullptr, nullptr};
  for (int k = 1; k < n_h2d; ++k) {
    if (!ctx->hsx[k - 1]) {
      ck(cudaStreamCreateWithFlags(&ctx->hsx[k - 1], cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&ctx->ev_hsx[k - 1], cudaEventDisableTiming), "event");
    }
    h2d[k] = ctx->hsx[k - 1];
  }
  ck(cudaEventRecord(ctx->ev_start, ctx->cs), "event");
  ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_start, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->ds, ctx->ev_start, 0), "wait");
  for (int k = 1; k < n_h2d; ++k) ck(cudaStreamWaitEvent(h2d[k], ctx->ev_start, 0), "wait");
  size_t rr = 0;
  // consecutive TR_MM contractions share one batched trace launch (CC_TR_BATCH=0: one each);
  // the batch is launched before any other op is issued, and its source events right after
  static const bool tr_batch = !(getenv("CC_TR_BATCH") && atoi(getenv("CC_TR_BATCH")) == 0);
  std::vector<const void*> ta, tb;
  std::vector<void*> tout;
  std::vector<size_t> tops;
  auto flush_tr = [&]() {
    if (tops.empty()) return;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (time_kernels) {
      ck(cudaEventCreate(&e0), "event");
      ck(cudaEventCreate(&e1), "event");
      ck(cudaEventRecord(e0, ctx->cs), "event");
    }
    ck(launch_trace_batch(ta.data(), tb.data(), tout.data(), int(tops.size()), g.Lt, g.N, ctx->trace_ws, ctx->cs),
       "TR_MM batch");
    ++nl;
    if (time_kernels) {
      ck(cudaEventRecord(e1, ctx->cs), "event");
      kev->push_back({e0, e1});
      kev_kind->push_back(CC_TR_MM);
    }
    for (size_t k : tops)
      if (ctx->pp.ops[k].source) ck(cudaEventRecord(ctx->events[k], ctx->cs), "event");
    ta.clear();
    tb.clear();
    tout.clear();
    tops.clear();
  };
  for (size_t i = 0; i < ctx->pp.ops.size(); ++i) {
    const PhysOp& op = ctx->pp.ops[i];
    if (op.stream == S_NONE) continue;
    if (tr_batch && op.kind == OP_CONTRACT && g.nodes[size_t(op.node)].op == CC_TR_MM) {
      const Node& n = g.nodes[size_t(op.node)];
      for (int32_t d : op.deps) ck(cudaStreamWaitEvent(ctx->cs, ctx->events[size_t(d)], 0), "wait");
      ta.push_back(op.loc_a == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.l)] : ctx->arena + op.off_a);
      tb.push_back(op.loc_b == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.r)] : ctx->arena + op.off_b);
      tout.push_back(ctx->roots + g.tree_of_root[size_t(op.node)] * g.Lt);
      tops.push_back(i);
      if (int(tops.size()) == trace_batch_max()) flush_tr();
      continue;
    }
    flush_tr();
    cudaStream_t s = st[op.stream];
    if (op.stream == S_H2D && n_h2d > 1) {
      s = h2d[rr++ % size_t(n_h2d)];
      for (int32_t d : op.same_deps) ck(cudaStreamWaitEvent(s, ctx->events[size_t(d)], 0), "wait");
    }
    for (int32_t d : op.deps) ck(cudaStreamWaitEvent(s, ctx->events[size_t(d)], 0), "wait");
    const Node& n = g.nodes[size_t(op.node)];
    switch (op.kind) {
      case OP_H2D: {
        const void* src;
        if (n.leaf()) {
          const char* h = static_cast<const char*>(ctx->leaf_host[size_t(op.node)]);
          if (!h) throw Error(CC_E_STATE, "leaf " + std::to_string(n.id) + " has no data (cc_set_leaf)");
          const int64_t per_t = n.op == CC_LEAF_M ? per_t_m : per_t_m * g.S * g.N;
          src = h + int64_t(ctx->t0) * per_t;
        } else {
          src = ctx->host_pool + op.host_off;
        }
        ck(cudaMemcpyAsync(ctx->arena + op.dev_off, src, size_t(op.bytes), cudaMemcpyHostToDevice, s), "H2D");
        break;
      }
      case OP_D2H:
        ck(cudaMemcpyAsync(ctx->host_pool + op.host_off, ctx->arena + op.dev_off, size_t(op.bytes),
                           cudaMemcpyDeviceToHost, s),
           "D2H");
        break;
      case OP_CONTRACT: {
        const void* a = op.loc_a == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.l)] : ctx->arena + op.off_a;
        const void* b = op.loc_b == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.r)] : ctx->arena + op.off_b;
        void* out = op.dev_off >= 0 ? ctx->arena + op.dev_off : nullptr;
        const int64_t slot = n.type == ROOT ? g.tree_of_root[size_t(op.node)] : -1;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (time_kernels) {
          ck(cudaEventCreate(&e0), "event");
          ck(cudaEventCreate(&e1), "event");
          ck(cudaEventRecord(e0, s), "event");
        }
        launch_contract(ctx, n, a, b, out, slot, &nl);
        if (time_kernels) {
          ck(cudaEventRecord(e1, s), "event");
          kev->push_back({e0, e1});
          kev_kind->push_back(n.op);
        }
        break;
      }
      default:
        break;
    }
    if (op.source) ck(cudaEventRecord(ctx->events[i], s), "event");
  }
  flush_tr();
  ck(launch_correlate(ctx->roots, ctx->corr, int64_t(g.corr_ids.size()), g.Lt, ctx->term_start, ctx->term_tree,
                      ctx->term_coef, ctx->cs),
     "correlate kernel");
  ++nl;
  for (int k = 1; k < n_h2d; ++k) {                 // join the extra H2D streams
    ck(cudaEventRecord(ctx->ev_hsx[k - 1], h2d[k]), "event");
    ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_hsx[k - 1], 0), "wait");
  }
  ck(cudaEventRecord(ctx->ev_h_end, ctx->hs), "event");
  ck(cudaEventRecord(ctx->ev_d_end, ctx->ds), "event");
  ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_h_end, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_d_end, 0), "wait");
  return nl;
}

// Replays only the contraction launches of one class (0: MM1/BM1/BB2, 1: TR_MM) of the
// current plan, in plan order, as a cached CUDA graph; requires a previous full execute
// (operands are wherever the plan put them; outputs are overwritten).  stats->seconds is
// the device time of the whole replay, stats->n_kernels the launches of that class.
void kernel_only(cc_ctx* ctx, int cls, cc_exec_stats* stats) {
  if (!ctx->executed) throw Error(CC_E_STATE, "kernel-only replay needs a previous full cc_execute");
  const Dag& g = *ctx->dag;
  cudaGraphExec_t& gx = ctx->gexec_kind[cls];
  int nl = 0;
  double flops = 0, bytes = 0;
  for (const auto& op : ctx->pp.ops) {
    if (op.kind != OP_CONTRACT) continue;
    const Node& n = g.nodes[size_t(op.node)];
    if ((n.op == CC_TR_MM) != (cls == 1)) continue;
    ++nl;
    flops += node_flops(n, g.Lt, g.N, g.S);
    bytes += node_hbm_bytes(n, g.Lt, g.N, g.S);
  }
  if (!gx) {
    cudaGraph_t graph;
    ck(cudaStreamBeginCapture(ctx->cs, cudaStreamCaptureModeThreadLocal), "graph capture");
    int launched = 0;
    try {
      for (const auto& op : ctx->pp.ops) {
        if (op.kind != OP_CONTRACT) continue;
        const Node& n = g.nodes[size_t(op.node)];
        if ((n.op == CC_TR_MM) != (cls == 1)) continue;
        const void* a = op.loc_a == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.l)] : ctx->arena + op.off_a;
        const void* b = op.loc_b == LOC_DEVLEAF ? ctx->leaf_dev[size_t(n.r)] : ctx->arena + op.off_b;
        if (!a || !b) throw Error(CC_E_STATE, "kernel-only replay: operand without a device address");
        void* out = op.dev_off >= 0 ? ctx->arena + op.dev_off : nullptr;
        const int64_t slot = n.type == ROOT ? g.tree_of_root[size_t(op.node)] : -1;
        launch_contract(ctx, n, a, b, out, slot, &launched);
      }
    } catch (...) {
      cudaStreamEndCapture(ctx->cs, &graph);
      throw;
    }
    ck(cudaStreamEndCapture(ctx->cs, &graph), "graph capture");
    ck(cudaGraphInstantiate(&gx, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
  }
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  ck(cudaEventRecord(e0, ctx->cs), "event");
  ck(cudaGraphLaunch(gx, ctx->cs), "graph launch");
  ck(cudaEventRecord(e1, ctx->cs), "event");
  ck(cudaEventSynchronize(e1), "kernel-only replay");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->seconds = ms * 1e-3;
    stats->flops = flops;
    stats->hbm_bytes = bytes;
    stats->n_kernels = nl;
  }
}

void execute(cc_ctx* ctx, int32_t flags, bool blocking, cc_exec_stats* stats) {
  ctx->need_device();
  if (!ctx->scheduled) throw Error(CC_E_STATE, "cc_execute before cc_schedule");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaEvent_t t_begin, t_end;
  ck(cudaEventCreate(&t_begin), "event");
  ck(cudaEventCreate(&t_end), "event");
  ck(cudaEventRecord(t_begin, ctx->cs), "event");   // before any preparation: seconds = time to solution
  // A plan that is about to be (re)built starts with host-leaf H2Ds into an empty pool: next-fit
  // places them back to back from offset 0, so up to 4 of those copies start before the
  // physical plan exists (prepare_dataflow checks the placement and adds the flag writes;
  // dataflow executor only; CC_PRECOPY=0 disables).
  ctx->pre_n = 0;
  std::vector<int64_t> pre_off;
  if (!(getenv("CC_PRECOPY") && atoi(getenv("CC_PRECOPY")) == 0) && !ctx->phys_valid &&
      !(flags & (2 | 4 | 8 | 16 | 64 | 128)) && !getenv("CC_H2D_CHUNK_MB") &&
      !getenv("CC_H2D_TAIL") && !(getenv("CC_EARLY_COPIES") && atoi(getenv("CC_EARLY_COPIES")) == 0)) {
    const Dag& g0 = *ctx->dag;
    int64_t off = 0;
    for (size_t j = 0; j < ctx->lp.ops.size() && j < 4; ++j) {
      const auto& lop = ctx->lp.ops[j];
      if (lop.kind != OP_H2D) break;
      const int32_t u = lop.node;
      const Node& n0 = g0.nodes[size_t(u)];
      if (!n0.leaf() || ctx->leaf_dev[size_t(u)] || !ctx->leaf_host[size_t(u)]) break;
      if (!ctx->ev_precopy) ck(cudaEventCreateWithFlags(&ctx->ev_precopy, cudaEventDisableTiming), "event");
      if (j == 0) {
        ck(cudaEventRecord(ctx->ev_precopy, ctx->cs), "event");   // after all earlier work on cs
        ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_precopy, 0), "wait");
      }
      const int64_t per_t_m = 16LL * g0.N * g0.N;
      const int64_t per_t = n0.op == CC_LEAF_M ? per_t_m : per_t_m * g0.S * g0.N;
      const char* src = static_cast<const char*>(ctx->leaf_host[size_t(u)]) + int64_t(ctx->t0) * per_t;
      ck(cudaMemcpyAsync(ctx->arena + off, src, size_t(n0.size), cudaMemcpyHostToDevice, ctx->hs), "H2D");
      pre_off.push_back(off);
      off += round_up(n0.size, ALIGN);
    }
    if (!pre_off.empty()) {
      ck(cudaEventRecord(ctx->ev_precopy, ctx->hs), "event");
      ctx->pre_n = int(pre_off.size());
    }
  }
  prepare_phys(ctx);
  for (int j = 0; j < ctx->pre_n; ++j) {
    const bool ok = size_t(j) < ctx->pp.ops.size() && ctx->pp.ops[size_t(j)].kind == OP_H2D &&
                    ctx->pp.ops[size_t(j)].dev_off == pre_off[size_t(j)] &&
                    ctx->pp.ops[size_t(j)].node == ctx->lp.ops[size_t(j)].node;
    if (!ok) {
      // placement differs: the early path copies those leaves again; nothing may touch the
      // pre-copied ranges on the compute stream before the stray copies are done
      ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_precopy, 0), "wait");
      ctx->pre_n = 0;
      break;
    }
  }
  if (flags & 128) {
    // CC_EXEC_AUTO: the Ozaki engine (bit 6) where it measured faster than the dataflow worker
    // (DESIGN §7): GEMMs with N >= 256, or baryon GEMMs with N >= 128
    const Dag& gd = *ctx->dag;
    bool gemm = false, baryon = false;
    for (const auto& n : gd.nodes) {
      gemm |= n.op == CC_MM1 || n.op == CC_BM1 || n.op == CC_BB2;
      baryon |= n.op == CC_BM1 || n.op == CC_BB2;
    }
    if (gemm && (gd.N >= 256 || (baryon && gd.N >= 128))) flags |= 64;
    flags &= ~128;
  }
  ctx->mm1_ozaki = (flags & 64) != 0;
  if (ctx->mm1_ozaki) oz_cache_reset(ctx);
  if (flags & 12) {
    kernel_only(ctx, (flags & 4) ? 0 : 1, stats);
    return;
  }
  const bool use_graph = (flags & 1) != 0;
  const bool legacy = (flags & 16) != 0 || (flags & 2) != 0 || (flags & 64) != 0;
  const bool time_kernels = (flags & 2) != 0 && !use_graph;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;
  std::vector<int> kev_kind;
  if (!legacy) {
    prepare_dataflow(ctx, getenv("CC_EARLY_COPIES") ? atoi(getenv("CC_EARLY_COPIES")) != 0 : true);
    const bool prof = (flags & 32) != 0;
    if (prof && !ctx->df_prof) {
      const int64_t n = ctx->df_gemm_items + ctx->df_trace_items + 2 * ctx->num_sms;
      ck(cudaMalloc(reinterpret_cast<void**>(&ctx->df_prof), size_t(n) * 64), "profile buffer");
      ck(cudaMemsetAsync(ctx->df_prof, 0, size_t(n) * 64, ctx->cs), "profile buffer");
    }
    ctx->df_gemm.prof = prof ? ctx->df_prof : nullptr;
    ctx->df_gemm.prof_t = prof ? ctx->df_prof + 8 * ctx->df_gemm_items : nullptr;
    ctx->df_gemm.prof_sm = prof ? reinterpret_cast<long long*>(ctx->df_prof + 8 * (ctx->df_gemm_items + ctx->df_trace_items)) : nullptr;
    if (prof && ctx->gexec_df) {
      cudaGraphExecDestroy(ctx->gexec_df);
      ctx->gexec_df = nullptr;
    }
  }
  if (!legacy) {
    if (use_graph && ctx->df_copies.empty()) {
      if (!ctx->gexec_df) {
        cudaGraph_t graph;
        ck(cudaStreamBeginCapture(ctx->cs, cudaStreamCaptureModeThreadLocal), "graph capture");
        try {
          ctx->last_n_kernels = issue_dataflow(ctx);
        } catch (...) {
          cudaStreamEndCapture(ctx->cs, &graph);
          throw;
        }
        ck(cudaStreamEndCapture(ctx->cs, &graph), "graph capture");
        ck(cudaGraphInstantiate(&ctx->gexec_df, graph, 0), "graph instantiate");
        cudaGraphDestroy(graph);
      }
      ck(cudaGraphLaunch(ctx->gexec_df, ctx->cs), "graph launch");
    } else {
      ctx->last_n_kernels = issue_dataflow(ctx, blocking);
    }
  } else if (use_graph) {
    if (!ctx->gexec) {
      cudaGraph_t graph;
      ck(cudaStreamBeginCapture(ctx->cs, cudaStreamCaptureModeThreadLocal), "graph capture");
      try {
        ctx->last_n_kernels = issue(ctx, false, nullptr, nullptr);
      } catch (...) {
        cudaStreamEndCapture(ctx->cs, &graph);
        throw;
      }
      ck(cudaStreamEndCapture(ctx->cs, &graph), "graph capture");
      ck(cudaGraphInstantiate(&ctx->gexec, graph, 0), "graph instantiate");
      cudaGraphDestroy(graph);
    }
    ck(cudaGraphLaunch(ctx->gexec, ctx->cs), "graph launch");
  } else {
    ctx->last_n_kernels = issue(ctx, time_kernels, &kev, &kev_kind);
  }
  ck(cudaEventRecord(t_end, ctx->cs), "event");
  ctx->executed = true;
  if (blocking) {
    ck(cudaEventSynchronize(t_end), "execute");
    ck(cudaGetLastError(), "execute");
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    if (blocking) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, t_begin, t_end), "elapsed");
      stats->seconds = ms * 1e-3;
      if (ctx->copy_timed && !ctx->df_copies.empty()) {
        float mh = 0, md = 0;
        ck(cudaEventElapsedTime(&mh, t_begin, ctx->ev_copy_h), "elapsed");
        ck(cudaEventElapsedTime(&md, t_begin, ctx->ev_copy_d), "elapsed");
        stats->copy_seconds = std::max(mh, md) * 1e-3;
      }
    }
    const Dag& g = *ctx->dag;
    for (const auto& op : ctx->pp.ops)
      if (op.kind == OP_CONTRACT) {
        stats->flops += node_flops(g.nodes[size_t(op.node)], g.Lt, g.N, g.S);
        stats->hbm_bytes += node_hbm_bytes(g.nodes[size_t(op.node)], g.Lt, g.N, g.S);
      }
    stats->h2d_bytes = ctx->pp.h2d_bytes;
    stats->d2h_bytes = ctx->pp.d2h_bytes;
    stats->n_kernels = ctx->last_n_kernels;
  }
  ctx->ktimes = KindTimes{};
  for (size_t i = 0; i < kev.size(); ++i) {
    float ms = 0;
    if (blocking) cudaEventElapsedTime(&ms, kev[i].first, kev[i].second);
    ctx->ktimes.seconds[kev_kind[i]] += ms * 1e-3;
    ctx->ktimes.count[kev_kind[i]] += 1;
    cudaEventDestroy(kev[i].first);
    cudaEventDestroy(kev[i].second);
  }
  if (stats) {
    double ks = 0;
    for (int k = 0; k < 8; ++k) ks += ctx->ktimes.seconds[k];
    stats->kernel_seconds = ks;
  }
  cudaEventDestroy(t_begin);
  cudaEventDestroy(t_end);
}

void ensure_ws(char*& ws, size_t& have, size_t bytes) {
  if (bytes <= have) return;
  if (ws) ck(cudaFree(ws), "cudaFree");
  ws = nullptr;
  have = 0;
  ck(cudaMalloc(reinterpret_cast<void**>(&ws), bytes), "workspace");
  ck(cudaMemset(ws, 0, bytes), "workspace");  // trace counters must start at zero
  ck(cudaDeviceSynchronize(), "workspace");   // (legacy-stream memset; kernels run on other streams)
  have = bytes;
}

}  // namespace

// ------------------------------------------------------------------------------------------
extern "C" {

const char* cc_version(void) { return CC_VERSION; }

const char* cc_last_error(const cc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

cc_status cc_create(cc_ctx** out, int device, void* dev_arena, size_t arena_bytes, void* compute_stream,
                    void* h2d_stream, void* d2h_stream) {
  cc_ctx* ctx = nullptr;
  if (!out) return CC_E_INVAL;
  *out = nullptr;
  try {
    ctx = new cc_ctx();
  } catch (...) {
    return CC_E_NOMEM;
  }
  API_BEGIN
  ctx->device = device;
  ctx->host_only = device < 0;
  *out = ctx;
  if (!ctx->host_only) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) throw Error(CC_E_CUDA, std::string("needs an sm_100 GPU (B200), found ") + prop.name);
    ctx->num_sms = prop.multiProcessorCount;
    ctx->arena = static_cast<char*>(dev_arena);
    ctx->arena_bytes = int64_t(arena_bytes);
    if (compute_stream) {
      ctx->cs = static_cast<cudaStream_t>(compute_stream);
      ctx->hs = static_cast<cudaStream_t>(h2d_stream);
      ctx->ds = static_cast<cudaStream_t>(d2h_stream);
      if (!ctx->hs || !ctx->ds) throw Error(CC_E_INVAL, "give all three streams or none");
    } else {
      ctx->own_streams = true;
      ck(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&ctx->hs, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&ctx->ds, cudaStreamNonBlocking), "stream");
    }
    for (cudaEvent_t* e : {&ctx->ev_start, &ctx->ev_end, &ctx->ev_h_end, &ctx->ev_d_end, &ctx->ev_pre, &ctx->ev_meta})
      ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    for (cudaEvent_t* e : {&ctx->ev_copy_h, &ctx->ev_copy_d}) ck(cudaEventCreate(e), "event");
    ck(zgemm_preload(), "kernel load");
    ck(trace_preload(), "kernel load");
    ck(df_preload(), "kernel load");
  }
  API_END
}

void cc_destroy(cc_ctx* ctx) { delete ctx; }

cc_status cc_load_dag(cc_ctx* ctx, const cc_dims* dims, const cc_node* nodes, int64_t n_nodes, const cc_tree* trees,
                      int64_t n_trees, const cc_term* terms, int64_t n_terms) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!dims || (n_nodes > 0 && !nodes) || (n_trees > 0 && !trees) || (n_terms > 0 && !terms) || n_nodes < 0 ||
      n_trees < 0 || n_terms < 0)
    throw Error(CC_E_INVAL, "null or negative DAG arrays");
  Input in;
  in.dims = *dims;
  in.nodes.assign(nodes, nodes + n_nodes);
  in.trees.assign(trees, trees + n_trees);
  in.terms.assign(terms, terms + n_terms);
  ctx->loaded = false;
  ctx->input = std::move(in);
  ctx->n_parts = 1;
  ctx->part = 0;
  rebuild_dag(ctx);
  ctx->loaded = true;
  API_END
}

cc_status cc_load_dag_file(cc_ctx* ctx, const char* path) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!path) throw Error(CC_E_INVAL, "null path");
  Input in = parse_text_file(path);
  ctx->loaded = false;
  ctx->input = std::move(in);
  ctx->n_parts = 1;
  ctx->part = 0;
  rebuild_dag(ctx);
  ctx->loaded = true;
  API_END
}

cc_status cc_dag_info(cc_ctx* ctx, cc_dag_stats* out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  if (!out) throw Error(CC_E_INVAL, "null output");
  *out = ctx->dag->stats();
  API_END
}

cc_status cc_partition(cc_ctx* ctx, int32_t n_parts, int32_t part, int32_t mode) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  if (n_parts < 1 || part < 0 || part >= n_parts || mode < 0 || mode > 1) throw Error(CC_E_INVAL, "bad partition");
  ctx->n_parts = n_parts;
  ctx->part = part;
  ctx->mode = mode;
  rebuild_dag(ctx);
  API_END
}

cc_status cc_part_trees(cc_ctx* ctx, int64_t* out, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  if (n_out) *n_out = int64_t(ctx->part_trees.size());
  if (out) {
    if (cap < int64_t(ctx->part_trees.size())) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    std::copy(ctx->part_trees.begin(), ctx->part_trees.end(), out);
  }
  API_END
}

cc_status cc_part_time_range(cc_ctx* ctx, int32_t* t0, int32_t* t1) {
  if (!ctx || !t0 || !t1) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  *t0 = ctx->t0;
  *t1 = ctx->t1;
  API_END
}

cc_status cc_schedule(cc_ctx* ctx, const cc_sched_cfg* cfg, int64_t* order_out, int64_t order_cap, int64_t* n_order,
                      cc_plan_stats* stats) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "cc_schedule before cc_load_dag");
  if (!cfg) throw Error(CC_E_INVAL, "null config");
  const Dag& g = *ctx->dag;
  ctx->scheduled = false;
  ctx->executed = false;
  ctx->release_phys();
  auto t0 = std::chrono::steady_clock::now();
  std::vector<int32_t> order;
  std::vector<int32_t> tree_order;
  if (cfg->algo == CC_SIBLING) {
    order = sibling_schedule(g);
  } else if (cfg->algo == CC_TREE) {
    TreeSchedule ts = tree_schedule(g);
    order = std::move(ts.order);
    tree_order = std::move(ts.tree_order);
  } else if (cfg->algo == CC_RSGS) {
    order = rsgs_schedule(g);
    tree_order = rsgs_tree_chain(g);
  } else if (cfg->algo == CC_GIVEN) {
    if (cfg->n_given < 0 || (cfg->n_given > 0 && !cfg->given_order)) throw Error(CC_E_INVAL, "bad given order");
    order.reserve(size_t(cfg->n_given));
    for (int64_t i = 0; i < cfg->n_given; ++i) order.push_back(g.idx(cfg->given_order[i]));
  } else {
    throw Error(CC_E_INVAL, "unknown scheduler");
  }
  auto t1 = std::chrono::steady_clock::now();
  check_order(g, order);
  ctx->mt = simulate_model(g, order);
  ctx->lp = lru_plan(g, order, cfg->cap_bytes, (cfg->flags & CC_EVICT_NEXT_USE) ? EVICT_NEXT_USE : EVICT_LRU);
  auto t2 = std::chrono::steady_clock::now();
  ctx->order = std::move(order);
  ctx->tree_order = std::move(tree_order);
  ctx->cap = cfg->cap_bytes;
  cc_plan_stats& s = ctx->stats;
  s = cc_plan_stats{};
  s.n_contr = g.n_contr;
  s.peak = ctx->lp.peak;
  s.transient_peak = ctx->lp.transient_peak;
  s.evictions = ctx->lp.evictions;
  s.h2d_count = ctx->lp.h2d_count;
  s.d2h_count = ctx->lp.d2h_count;
  s.h2d_bytes = ctx->lp.h2d_bytes;
  s.d2h_bytes = ctx->lp.d2h_bytes;
  s.host_peak_bytes = ctx->lp.host_peak;
  s.model_peak = ctx->mt.peak;
  s.model_transient_peak = ctx->mt.transient_peak;
  s.sched_seconds = std::chrono::duration<double>(t1 - t0).count();
  s.plan_seconds = std::chrono::duration<double>(t2 - t1).count();
  ctx->scheduled = true;
  if (n_order) *n_order = int64_t(ctx->order.size());
  if (order_out) {
    if (order_cap < int64_t(ctx->order.size())) throw Error(CC_E_BUFFER_TOO_SMALL, "order buffer too small");
    for (size_t i = 0; i < ctx->order.size(); ++i) order_out[i] = g.nodes[size_t(ctx->order[i])].id;
  }
  if (stats) *stats = s;
  API_END
}

cc_status cc_memory_trace(cc_ctx* ctx, int64_t* m_out, int64_t* transient_out, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->scheduled) throw Error(CC_E_STATE, "no schedule");
  const int64_t n = int64_t(ctx->mt.transient.size());
  if (n_out) *n_out = n;
  if (m_out) {
    if (cap < n + 1) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    std::copy(ctx->mt.M.begin(), ctx->mt.M.end(), m_out);
  }
  if (transient_out) {
    if (cap < n) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    std::copy(ctx->mt.transient.begin(), ctx->mt.transient.end(), transient_out);
  }
  API_END
}

cc_status cc_plan_ops(cc_ctx* ctx, cc_plan_op* out, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->scheduled) throw Error(CC_E_STATE, "no schedule");
  const auto& ops = ctx->lp.ops;
  if (n_out) *n_out = int64_t(ops.size());
  if (out) {
    if (cap < int64_t(ops.size())) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    const bool phys = ctx->phys_valid;
    for (size_t i = 0; i < ops.size(); ++i) {
      const Node& n = ctx->dag->nodes[size_t(ops[i].node)];
      out[i] = cc_plan_op{ops[i].kind, 0, n.id, n.size, phys ? ctx->pp.ops[i].dev_off : -1};
    }
  }
  API_END
}

cc_status cc_tree_order(cc_ctx* ctx, int64_t* out, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->scheduled) throw Error(CC_E_STATE, "no schedule");
  if (n_out) *n_out = int64_t(ctx->tree_order.size());
  if (out) {
    if (cap < int64_t(ctx->tree_order.size())) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    for (size_t i = 0; i < ctx->tree_order.size(); ++i) out[i] = ctx->dag->trees[size_t(ctx->tree_order[i])].tree_id;
  }
  API_END
}

cc_status cc_plan_dump(cc_ctx* ctx, const char* csv_path) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->scheduled) throw Error(CC_E_STATE, "no schedule");
  std::ofstream f(csv_path);
  if (!f) throw Error(CC_E_INVAL, "cannot write " + std::string(csv_path ? csv_path : "(null)"));
  static const char* kinds[5] = {"H2D", "D2H", "DROP", "CONTRACT", "FREE"};
  f << "step,op,node,bytes,offset,device_used\n";
  int64_t step = 0;
  for (size_t i = 0; i < ctx->lp.ops.size(); ++i) {
    const auto& op = ctx->lp.ops[i];
    const Node& n = ctx->dag->nodes[size_t(op.node)];
    if (op.kind == OP_CONTRACT) ++step;
    f << step << ',' << kinds[op.kind] << ',' << n.id << ',' << n.size << ','
      << (ctx->phys_valid ? ctx->pp.ops[i].dev_off : -1) << ',' << ctx->lp.used[size_t(step)] << '\n';
  }
  API_END
}

cc_status cc_set_leaf(cc_ctx* ctx, int64_t leaf_id, const void* host, size_t bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  const Dag& g = *ctx->dag;
  auto it = g.index.find(leaf_id);
  if (it == g.index.end()) {
    // a leaf of another TREES part: accepted and ignored
    for (const auto& n : ctx->input.nodes)
      if (n.id == leaf_id) return CC_OK;
    throw Error(CC_E_UNKNOWN_NODE, "unknown leaf " + std::to_string(leaf_id));
  }
  const Node& n = g.nodes[size_t(it->second)];
  if (!n.leaf()) throw Error(CC_E_INVAL, "node " + std::to_string(leaf_id) + " is not a leaf");
  const int64_t full = tensor_bytes(n.op, ctx->input.dims.Lt, g.N, g.S);
  if (int64_t(bytes) != full) throw Error(CC_E_INVAL, "leaf " + std::to_string(leaf_id) + ": expected " + std::to_string(full) + " bytes");
  if (!host) throw Error(CC_E_INVAL, "null host pointer");
  const bool was_dev = ctx->leaf_dev[size_t(it->second)] != nullptr;
  ctx->leaf_host[size_t(it->second)] = host;
  ctx->leaf_dev[size_t(it->second)] = nullptr;
  if (was_dev) {
    ctx->phys_valid = false;
    ctx->release_graph();
  }
  ctx->release_graph();  // host pointers are baked into a captured graph
  API_END
}

cc_status cc_set_leaf_device(cc_ctx* ctx, int64_t leaf_id, const void* dev, size_t bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  const Dag& g = *ctx->dag;
  auto it = g.index.find(leaf_id);
  if (it == g.index.end()) {
    for (const auto& n : ctx->input.nodes)
      if (n.id == leaf_id) return CC_OK;
    throw Error(CC_E_UNKNOWN_NODE, "unknown leaf " + std::to_string(leaf_id));
  }
  const Node& n = g.nodes[size_t(it->second)];
  if (!n.leaf()) throw Error(CC_E_INVAL, "node " + std::to_string(leaf_id) + " is not a leaf");
  if (int64_t(bytes) != n.size) throw Error(CC_E_INVAL, "leaf " + std::to_string(leaf_id) + ": expected " + std::to_string(n.size) + " bytes");
  if (!dev) throw Error(CC_E_INVAL, "null device pointer");
  const bool was_dev = ctx->leaf_dev[size_t(it->second)] != nullptr;
  ctx->leaf_dev[size_t(it->second)] = dev;
  ctx->leaf_host[size_t(it->second)] = nullptr;
  if (!was_dev) ctx->phys_valid = false;
  ctx->release_graph();
  API_END
}

cc_status cc_execute(cc_ctx* ctx, int32_t flags, cc_exec_stats* stats) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  execute(ctx, flags, true, stats);
  API_END
}

cc_status cc_execute_async(cc_ctx* ctx, int32_t flags) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  execute(ctx, flags & 1, false, nullptr);
  API_END
}

cc_status cc_correlator(cc_ctx* ctx, int64_t corr_id, double* out, int32_t Lt) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!ctx->executed) throw Error(CC_E_STATE, "cc_correlator before cc_execute");
  const Dag& g = *ctx->dag;
  if (Lt != g.Lt) throw Error(CC_E_INVAL, "Lt must be the part's Lt (" + std::to_string(g.Lt) + ")");
  auto it = std::lower_bound(g.corr_ids.begin(), g.corr_ids.end(), corr_id);
  if (it == g.corr_ids.end() || *it != corr_id) throw Error(CC_E_UNKNOWN_NODE, "unknown correlator " + std::to_string(corr_id));
  const int64_t slot = it - g.corr_ids.begin();
  ck(cudaStreamSynchronize(ctx->cs), "sync");
  ck(cudaMemcpyAsync(out, ctx->corr + slot * g.Lt, size_t(g.Lt) * 16, cudaMemcpyDeviceToHost, ctx->cs), "correlator D2H");
  ck(cudaStreamSynchronize(ctx->cs), "correlator D2H");
  API_END
}

cc_status cc_root_value(cc_ctx* ctx, int64_t tree_id, double* out, int32_t Lt) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!ctx->executed) throw Error(CC_E_STATE, "cc_root_value before cc_execute");
  const Dag& g = *ctx->dag;
  if (Lt != g.Lt) throw Error(CC_E_INVAL, "Lt must be the part's Lt");
  int64_t slot = -1;
  for (size_t t = 0; t < g.trees.size(); ++t)
    if (g.trees[t].tree_id == tree_id) slot = int64_t(t);
  if (slot < 0) throw Error(CC_E_UNKNOWN_NODE, "unknown tree " + std::to_string(tree_id));
  ck(cudaStreamSynchronize(ctx->cs), "sync");
  ck(cudaMemcpyAsync(out, ctx->roots + slot * g.Lt, size_t(g.Lt) * 16, cudaMemcpyDeviceToHost, ctx->cs), "root D2H");
  ck(cudaStreamSynchronize(ctx->cs), "root D2H");
  API_END
}

cc_status cc_correlator_device_ptr(cc_ctx* ctx, void** dev_ptr, int64_t* n_corr, int64_t* corr_ids) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!ctx->executed) throw Error(CC_E_STATE, "before cc_execute");
  const Dag& g = *ctx->dag;
  if (dev_ptr) *dev_ptr = ctx->corr;
  if (n_corr) *n_corr = int64_t(g.corr_ids.size());
  if (corr_ids) std::copy(g.corr_ids.begin(), g.corr_ids.end(), corr_ids);
  API_END
}

cc_status cc_correlators(cc_ctx* ctx, double* out, int64_t cap) {
  if (!ctx || !out) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!ctx->executed) throw Error(CC_E_STATE, "before cc_execute");
  const Dag& g = *ctx->dag;
  const int64_t n = int64_t(g.corr_ids.size()) * g.Lt * 2;
  if (cap < n) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
  ck(cudaMemcpyAsync(out, ctx->corr, size_t(n) * 8, cudaMemcpyDeviceToHost, ctx->cs), "correlators D2H");
  ck(cudaStreamSynchronize(ctx->cs), "correlators D2H");
  API_END
}

cc_status cc_dataflow_state(cc_ctx* ctx, int64_t* out, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!ctx->df_valid) throw Error(CC_E_STATE, "no dataflow plan");
  const size_t n_int = (ctx->df_sync_bytes - 16) / 4;
  std::vector<char> buf(ctx->df_sync_bytes);
  cudaStream_t s;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  ck(cudaMemcpyAsync(buf.data(), ctx->df_sync_base, buf.size(), cudaMemcpyDeviceToHost, s), "state copy");
  ck(cudaStreamSynchronize(s), "state copy");
  cudaStreamDestroy(s);
  const int64_t n = 2 + int64_t(n_int);
  if (n_out) *n_out = n;
  if (out) {
    if (cap < n) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    const unsigned long long* h = reinterpret_cast<const unsigned long long*>(buf.data());
    out[0] = int64_t(h[0]);
    out[1] = int64_t(h[1]);
    const int* sy = reinterpret_cast<const int*>(buf.data() + 16);
    for (size_t i = 0; i < n_int; ++i) out[2 + i] = sy[i];
  }
  API_END
}

cc_status cc_dataflow_profile(cc_ctx* ctx, uint64_t* out, int64_t cap, int64_t* n_gemm, int64_t* n_trace) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!ctx->df_prof) throw Error(CC_E_STATE, "no profiled dataflow execute (flags bit 5)");
  const int64_t n = ctx->df_gemm_items + ctx->df_trace_items + 2 * ctx->num_sms;
  if (n_gemm) *n_gemm = ctx->df_gemm_items;
  if (n_trace) *n_trace = ctx->df_trace_items;
  if (out) {
    if (cap < 8 * n) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    ck(cudaMemcpy(out, ctx->df_prof, size_t(n) * 64, cudaMemcpyDeviceToHost), "profile copy");
  }
  API_END
}

cc_status cc_kernel_times(cc_ctx* ctx, double* seconds, int64_t* counts) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  for (int k = 0; k < 8; ++k) {
    if (seconds) seconds[k] = ctx->ktimes.seconds[k];
    if (counts) counts[k] = ctx->ktimes.count[k];
  }
  API_END
}

static cc_status direct_gemm(cc_ctx* ctx, int op, const void* A, const void* B, void* C, int32_t Lt, int32_t N,
                             int32_t S) {
  API_BEGIN
  ctx->need_device();
  if (!A || !B || !C || Lt <= 0 || N <= 0 || S <= 0) throw Error(CC_E_INVAL, "bad kernel arguments");
  ZgemmProblem p = problem_for(op, Lt, N, S, A, B, C);
  ensure_ws(ctx->direct_ws, ctx->direct_ws_bytes, std::max<size_t>(zgemm_workspace_bytes(p, ctx->num_sms), 256));
  int nl = 0;
  ck(launch_zgemm(p, ctx->direct_ws, ctx->direct_ws_bytes, ctx->num_sms, ctx->cs, &nl), "contraction kernel");
  API_END
}

cc_status cc_mm1(cc_ctx* ctx, const void* A, const void* B, void* C, int32_t Lt, int32_t N) {
  if (!ctx) return CC_E_INVAL;
  return direct_gemm(ctx, CC_MM1, A, B, C, Lt, N, 1);
}
cc_status cc_bm1(cc_ctx* ctx, const void* A, const void* M, void* C, int32_t Lt, int32_t N, int32_t S) {
  if (!ctx) return CC_E_INVAL;
  return direct_gemm(ctx, CC_BM1, A, M, C, Lt, N, S);
}
cc_status cc_bb2(cc_ctx* ctx, const void* A, const void* B, void* C, int32_t Lt, int32_t N, int32_t S) {
  if (!ctx) return CC_E_INVAL;
  return direct_gemm(ctx, CC_BB2, A, B, C, Lt, N, S);
}
cc_status cc_tr_mm(cc_ctx* ctx, const void* A, const void* B, void* c, int32_t Lt, int32_t N) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!A || !B || !c || Lt <= 0 || N <= 0) throw Error(CC_E_INVAL, "bad kernel arguments");
  ensure_ws(ctx->direct_tr_ws, ctx->direct_tr_ws_bytes, trace_workspace_bytes(Lt, N));
  // counters must be zero; a previous direct call with another Lt may have left partials there
  ck(cudaMemsetAsync(ctx->direct_tr_ws, 0, size_t(Lt) * 4, ctx->cs), "memset");
  ck(launch_trace(A, B, c, Lt, N, ctx->direct_tr_ws, ctx->cs), "TR_MM kernel");
  API_END
}

size_t cc_gemm_ozaki_workspace_bytes(int32_t op, int32_t Lt, int32_t N, int32_t S, int32_t n_slices) {
  if ((op != CC_MM1 && op != CC_BM1 && op != CC_BB2) || Lt <= 0 || N <= 0 || S <= 0 || n_slices < 4 || n_slices > 7)
    return 0;
  return ozaki_workspace_bytes(problem_for(op, Lt, N, op == CC_MM1 ? 1 : S, nullptr, nullptr, nullptr), n_slices, Lt);
}

cc_status cc_gemm_ozaki(cc_ctx* ctx, int32_t op, const void* A, const void* B, void* C, int32_t Lt, int32_t N,
                        int32_t S, int32_t n_slices, void* workspace, size_t workspace_bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if ((op != CC_MM1 && op != CC_BM1 && op != CC_BB2) || !A || !B || !C || !workspace || Lt <= 0 || N <= 0 || S <= 0 ||
      n_slices < 4 || n_slices > 7)
    throw Error(CC_E_INVAL, "bad kernel arguments");
  const ZgemmProblem q = problem_for(op, Lt, N, op == CC_MM1 ? 1 : S, A, B, C);
  if (workspace_bytes < ozaki_workspace_bytes(q, n_slices, 1)) throw Error(CC_E_BUFFER_TOO_SMALL, "ozaki workspace too small");
  ck(launch_ozaki_gemm(q, n_slices, workspace, workspace_bytes, ctx->cs), "Ozaki GEMM");
  API_END
}

size_t cc_mm1_ozaki_workspace_bytes(int32_t Lt, int32_t N, int32_t n_slices) {
  if (Lt <= 0 || N <= 0 || N > 8192 || n_slices < 4 || n_slices > 7) return 0;
  return ozaki_mm1_workspace_bytes(Lt, N, n_slices);
}

cc_status cc_mm1_ozaki(cc_ctx* ctx, const void* A, const void* B, void* C, int32_t Lt, int32_t N, int32_t n_slices,
                       void* workspace, size_t workspace_bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!A || !B || !C || !workspace || Lt <= 0 || N <= 0 || N > 8192 || n_slices < 4 || n_slices > 7)
    throw Error(CC_E_INVAL, "bad kernel arguments");
  if (workspace_bytes < ozaki_mm1_workspace_bytes(Lt, N, n_slices))
    throw Error(CC_E_BUFFER_TOO_SMALL, "ozaki workspace too small");
  ck(launch_ozaki_mm1(A, B, C, Lt, N, n_slices, workspace, workspace_bytes, ctx->cs), "Ozaki MM1");
  API_END
}

cc_status cc_i8gemm_tn(cc_ctx* ctx, const int8_t* A, const int8_t* B, int32_t* C, int32_t M, int32_t Nn, int32_t K) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!A || !B || !C || M <= 0 || Nn <= 0 || K <= 0 || M % 128 || Nn % 192 || K % 64)
    throw Error(CC_E_INVAL, "bad kernel arguments (M % 128, Nn % 192, K % 64)");
  ck(launch_i8gemm_tn(A, B, C, M, Nn, K, ctx->cs), "int8 tcgen05 GEMM");
  API_END
}

cc_status cc_fill_synthetic(cc_ctx* ctx, void* dev, int64_t n, uint64_t seed, int64_t leaf_id, int64_t e0, int32_t mode,
                            double sigma) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!dev || n < 0 || e0 < 0 || mode < 0 || mode > 1) throw Error(CC_E_INVAL, "bad arguments");
  ck(launch_fill_synthetic(dev, n, seed, leaf_id, e0, mode, sigma, ctx->cs), "fill kernel");
  API_END
}

size_t cc_scratch_bytes(int32_t Lt, int32_t N, int32_t S) {
  // upper bound of prepare_phys's scratch for DAGs with up to 2^16 trees/terms/correlators
  size_t ws = 0;
  for (int op : {int(CC_MM1), int(CC_BM1), int(CC_BB2)})
    ws = std::max(ws, zgemm_workspace_bytes(problem_for(op, Lt, N, S, nullptr, nullptr, nullptr), 148));
  return ws + trace_workspace_bytes(Lt, N) + size_t(Lt) * 16 * 3 * 65536 + (size_t(16) << 20);
}

}  // extern "C"
