// Scratch layout and physical placement of a plan in the caller's arena.
#include "internal.hpp"

namespace ccx {

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
    // TREES (mode 1), or GRID (mode 2): TREES part part / n_time_parts, TIME part part % n_time_parts
    const int32_t nt = ctx->mode == 2 ? ctx->n_time_parts : 1;
    const int32_t pt = ctx->part / nt, ptm = ctx->part % nt;
    ctx->t0 = int32_t(int64_t(ptm) * Lt / nt);
    ctx->t1 = int32_t(int64_t(ptm + 1) * Lt / nt);
    if (ctx->t1 <= ctx->t0) throw Error(CC_E_INVAL, "GRID partition: part has no time slices");
    Dag full(ctx->input);
    std::vector<int32_t> parts = tree_parts(full, ctx->n_parts, nullptr);
    std::vector<int64_t> keep;
    for (size_t t = 0; t < full.trees.size(); ++t)
      if (parts[t] == pt) keep.push_back(full.trees[t].tree_id);
    if (keep.empty()) throw Error(CC_E_INVAL, "TREES partition: part has no trees");
    ctx->dag = std::make_unique<Dag>(ctx->input, nt > 1 ? ctx->t1 - ctx->t0 : 0, &keep);
    ctx->part_trees = keep;
  }
  const size_t n = ctx->dag->nodes.size();
  ctx->leaf_host.assign(n, nullptr);
  ctx->leaf_dev.assign(n, nullptr);
  ctx->leaf_peer.assign(n, nullptr);
  ctx->peer_home.assign(n, 0);
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
  } else if (op == CC_BB2) {
    p.M = N; p.Nn = N; p.Kin = N * N; p.Ko = S;
    p.lda = N * N; p.sAo = N * N * N; p.sAb = S * N * N * N;
    p.ldb = N; p.sBo = N * N * N; p.sBb = S * N * N * N;
    p.ldc = N; p.sCb = N * N;
  } else if (op == CC_BB1) {
    // T[t,(i,j),(l,m)] = sum_{s,k} A[t,s,(i,j),k] B[t,s,k,(l,m)]: M = N^2, Nn = N^2, K = (s, k)
    p.M = N * N; p.Nn = N * N; p.Kin = N; p.Ko = S;
    p.lda = N; p.sAo = N * N * N; p.sAb = S * N * N * N;
    p.ldb = N * N; p.sBo = N * N * N; p.sBb = S * N * N * N;
    p.ldc = N * N; p.sCb = N * N * N * N;
  } else {  // CC_BT2
    // C[t,(s,m),(i,j)] = sum_{(k,l)} A[t,(s,m),(k,l)] X[t,(k,l),(i,j)]: M = S N, Nn = N^2, K = N^2
    p.M = S * N; p.Nn = N * N; p.Kin = N * N; p.Ko = 1;
    p.lda = N * N; p.sAo = 0; p.sAb = S * N * N * N;
    p.ldb = N * N; p.sBo = 0; p.sBb = N * N * N * N;
    p.ldc = N * N; p.sCb = S * N * N * N;
  }
  return p;
}


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
int64_t df_trace_pieces(const TraceShape& sh) {
  constexpr int64_t units = 16;
  const int64_t nb = (sh.N + 31) / 32, U = int64_t(sh.G) * nb * nb;
  return std::max<int64_t>(1, (U + units - 1) / units);
}

// Byte sizes of the arena scratch regions (top of the arena, outside the logical pool; reading
// E-7) for the loaded DAG; also sets the dataflow ring slot sizes.
ScratchSizes scratch_sizes(cc_ctx* ctx) {
  const Dag& g = *ctx->dag;
  const int64_t Lt = g.Lt, N = g.N, S = g.S;
  ScratchSizes z;
  // scratch layout
  size_t gemm_ws = 0;
  bool has[CC_N_OPS] = {false};
  for (const auto& n : g.nodes) has[n.op] = true;
  for (int op : GEMM_OPS)
    if (has[op]) gemm_ws = std::max(gemm_ws, zgemm_workspace_bytes(problem_for(op, Lt, N, S, nullptr, nullptr, nullptr), ctx->num_sms));
  // Ozaki engine (execute flags bit 6): workspace for batches of time slices that fit in
  // max(one slice, arena / 16)
  for (int op : GEMM_OPS) {
    if (!has[op]) continue;
    const ZgemmProblem q = problem_for(op, Lt, N, S, nullptr, nullptr, nullptr);
    const size_t lim = std::max(ozaki_workspace_bytes(q, ctx->opt.ozaki_slices, 1), size_t(ctx->arena_bytes / 16));
    int64_t bt = Lt;
    while (bt > 1 && ozaki_workspace_bytes(q, ctx->opt.ozaki_slices, bt) > lim) bt = (bt + 1) / 2;
    gemm_ws = std::max(gemm_ws, ozaki_workspace_bytes(q, ctx->opt.ozaki_slices, bt));
  }
  // Ozaki leaf-form cache: one form per (leaf, op kind, side) read by a GEMM op; reserved
  // when it takes at most 1/8 of the arena (else the cache uses whatever pool space the plan
  // leaves free)
  int64_t sz_ozc = 0;
  {
    std::vector<std::array<char, 2 * OZ_KINDS>> role(g.nodes.size(), std::array<char, 2 * OZ_KINDS>{});
    for (const auto& n : g.nodes)
      if (is_gemm_kind(n.op)) {
        if (g.nodes[size_t(n.l)].leaf()) role[size_t(n.l)][size_t(2 * oz_kind(n.op))] = 1;
        if (g.nodes[size_t(n.r)].leaf()) role[size_t(n.r)][size_t(2 * oz_kind(n.op) + 1)] = 1;
      }
    int64_t fsz[2 * OZ_KINDS] = {0};
    for (int op : GEMM_OPS) {
      if (!has[op]) continue;
      const ZgemmProblem q = problem_for(op, Lt, N, S, nullptr, nullptr, nullptr);
      fsz[2 * oz_kind(op)] = round_up(int64_t(ozaki_form_bytes(q, ctx->opt.ozaki_slices, false)), ALIGN);
      fsz[2 * oz_kind(op) + 1] = round_up(int64_t(ozaki_form_bytes(q, ctx->opt.ozaki_slices, true)), ALIGN);
    }
    for (const auto& r : role)
      for (int k = 0; k < 2 * OZ_KINDS; ++k) sz_ozc += r[size_t(k)] ? fsz[k] : 0;
    if (sz_ozc > ctx->arena_bytes / 8) sz_ozc = 0;
  }
  size_t trace_ws = 0;
  for (int op : TRACE_OPS)
    if (has[op] || op == CC_TR_MM) trace_ws = std::max(trace_ws, trace_workspace_bytes(Lt, trace_shape(op, N, S)));
  const int64_t n_trees = int64_t(g.trees.size()), n_corr = int64_t(g.corr_ids.size()), n_terms = int64_t(g.terms.size());
  z.sz_gemm = round_up(int64_t(gemm_ws), ALIGN);
  z.sz_trace = round_up(int64_t(trace_ws), ALIGN);
  z.sz_roots = round_up(n_trees * Lt * 16, ALIGN);
  z.sz_corr = round_up(std::max<int64_t>(n_corr, 1) * Lt * 16, ALIGN);
  z.sz_ts = round_up((n_corr + 1) * 4, ALIGN);
  z.sz_tt = round_up(std::max<int64_t>(n_terms, 1) * 4, ALIGN);
  z.sz_tc = round_up(std::max<int64_t>(n_terms, 1) * 16, ALIGN);
  // dataflow workspaces: rings of chunk-partial slots (GEMM ops split in k) and of trace
  // partial slots (per-op tickets and [Lt][P] partials)
  ctx->df_chunk_slot = ctx->df_chunk_cnt_slot = 0;
  for (int op : GEMM_OPS) {
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
  int64_t pieces = 1;
  for (int op : TRACE_OPS)
    if (has[op]) pieces = std::max(pieces, df_trace_pieces(trace_shape(op, N, S)));
  ctx->df_trace_slot = round_up(Lt * pieces * 16, ALIGN) + round_up(Lt * 4, ALIGN);
  z.sz_df_chunk = DF_CHUNK_RING * (ctx->df_chunk_slot + ctx->df_chunk_cnt_slot);
  z.sz_df_trace = DF_TRACE_RING * ctx->df_trace_slot;
  z.sz_ozc = sz_ozc;
  z.total = z.sz_gemm + z.sz_trace + z.sz_roots + z.sz_corr + z.sz_ts + z.sz_tt + z.sz_tc + z.sz_df_chunk + z.sz_df_trace + z.sz_ozc;
  return z;
}

// Sets up scratch (kernel workspace, roots, correlators, term tables), the physical plan,
// events and the host pool.  Called lazily by cc_execute.
void prepare_phys(cc_ctx* ctx) {
  if (ctx->phys_valid) return;
  NvtxRange nv("cc prepare_phys");
  PhaseTimer pt("prepare_phys", (ctx->opt.debug & 2) != 0);
  ctx->release_phys();
  pt.lap("release");
  const Dag& g = *ctx->dag;
  if (g.abstract) throw Error(CC_E_STATE, "abstract DAG (leafX/OPX) can be scheduled, not executed");
  const int64_t Lt = g.Lt, N = g.N, S = g.S;
  const ScratchSizes z = scratch_sizes(ctx);
  const int64_t sz_gemm = z.sz_gemm, sz_trace = z.sz_trace, sz_roots = z.sz_roots, sz_corr = z.sz_corr, sz_ts = z.sz_ts,
                sz_tt = z.sz_tt, sz_tc = z.sz_tc, sz_df_chunk = z.sz_df_chunk, sz_df_trace = z.sz_df_trace, sz_ozc = z.sz_ozc,
                scratch = z.total;
  const size_t trace_ws = size_t(sz_trace);
  const int64_t n_corr = int64_t(g.corr_ids.size()), n_terms = int64_t(g.terms.size());
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
  int64_t phys_limit = pool;
  if (ctx->cap > 0) phys_limit = std::min(pool, round_up(ctx->cap + ctx->cap / 4, ALIGN));
  if (ctx->lp.p2p_out_count > 0 && !ctx->peer_tier)
    throw Error(CC_E_STATE, "the plan evicts to the peer tier and no region is set (cc_set_peer_tier)");
  for (size_t u = 0; u < g.nodes.size(); ++u)
    if (u < ctx->peer_home.size() && ctx->peer_home[u] && !on_dev[u] && !ctx->leaf_peer[u])
      throw Error(CC_E_STATE, "peer-homed leaf " + std::to_string(g.nodes[u].id) + " has no peer copy (cc_set_leaf_peer)");
  // Unbounded plans first try fixed leaf slots (every leaf copy then lands in memory no earlier
  // op touched, so all of them stream ahead at full PCIe rate instead of waiting, in plan
  // order, for intermediates to free their space); a capped plan keeps its footprint.
  bool placed = false;
  if (ctx->cap <= 0 && ctx->opt.leaf_slots) {
    try {
      ctx->pp = build_phys(g, ctx->lp, on_dev, phys_limit, ALIGN, RangeAlloc::NEXT_FIT, ctx->peer_tier_bytes, true);
      placed = true;
    } catch (const Error& e) {
      if (e.status != CC_E_NOMEM) throw;
    }
  }
  if (!placed) {
    try {
      ctx->pp = build_phys(g, ctx->lp, on_dev, phys_limit, ALIGN, RangeAlloc::NEXT_FIT, ctx->peer_tier_bytes);
    } catch (const Error& e) {
      if (e.status != CC_E_NOMEM) throw;
      try {
        ctx->pp = build_phys(g, ctx->lp, on_dev, pool, ALIGN, RangeAlloc::BEST_FIT, ctx->peer_tier_bytes);
      } catch (const Error& e2) {
        if (e2.status != CC_E_NOMEM) throw;
        // fragmentation: compact with device-to-device moves (op-by-op executor)
        ctx->pp = build_phys(g, ctx->lp, on_dev, pool, ALIGN, RangeAlloc::BEST_FIT, ctx->peer_tier_bytes, false, true);
      }
    }
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


}  // namespace ccx
