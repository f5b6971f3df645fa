// Op-by-op execution: one kernel launch per contraction (DMMA zgemm / trace kernels or the
// tcgen05 Ozaki engine), event edges between the three streams; kernel-only replays.
#include "internal.hpp"

namespace ccx {

// Resets the Ozaki leaf-form cache for one execute (or one kernel-only capture): the free
// pool range above the plan's high water, below any dataflow metadata / sync area placed at
// the top of the pool.  Option ozaki_leaf_cache = 0 disables it.
void oz_cache_reset(cc_ctx* ctx) {
  const size_t n = ctx->dag->nodes.size();
  for (int k = 0; k < 2 * OZ_KINDS; ++k) {
    ctx->oz.form[k].assign(n, OzakiForm{nullptr, nullptr});
    ctx->oz.have[k].assign(n, 0);
  }
  int64_t end = ctx->pool_bytes;
  if (ctx->df_sync_base) end = std::min<int64_t>(end, ctx->df_sync_base - ctx->arena);
  if (ctx->df_meta && !ctx->df_meta_owned) end = std::min<int64_t>(end, ctx->df_meta - ctx->arena);
  if (ctx->df_fpart && !ctx->df_fpart_owned) end = std::min<int64_t>(end, reinterpret_cast<char*>(ctx->df_fpart) - ctx->arena);
  const bool off = ctx->opt.ozaki_leaf_cache == 0;
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
  const int64_t bytes = round_up(int64_t(ozaki_form_bytes(q, ctx->opt.ozaki_slices, as_b)), ALIGN);
  if (ctx->oz.off + bytes > ctx->oz.end) return nullptr;
  ck(launch_ozaki_form(q, ctx->opt.ozaki_slices, as_b, ctx->arena + ctx->oz.off, &ctx->oz.form[k][size_t(u)], ctx->cs),
     "Ozaki leaf split");
  ctx->oz.off += bytes;
  ctx->oz.have[k][size_t(u)] = 1;
  return &ctx->oz.form[k][size_t(u)];
}

void launch_contract(cc_ctx* ctx, const Node& n, const void* a, const void* b, void* out, int64_t root_slot,
                     int* nl) {
  const Dag& g = *ctx->dag;
  if (is_root_kind(n.op)) {
    ck(launch_trace(a, b, ctx->roots + root_slot * g.Lt, g.Lt, trace_shape(n.op, g.N, g.S), ctx->trace_ws, ctx->cs),
       "contract-all kernel");
    ++*nl;
    return;
  }
  if (ctx->mm1_ozaki) {
    const ZgemmProblem q = problem_for(n.op, g.Lt, g.N, g.S, a, b, out);
    // forms only when the whole batch fits the workspace (else the engine splits per batch)
    const bool whole = ozaki_workspace_bytes(q, ctx->opt.ozaki_slices, g.Lt) <= ctx->gemm_ws_bytes;
    const OzakiForm* fa = whole ? oz_leaf_form(ctx, n.op, q, n.l, false) : nullptr;
    const OzakiForm* fb = whole ? oz_leaf_form(ctx, n.op, q, n.r, true) : nullptr;
    ck(launch_ozaki_gemm(q, ctx->opt.ozaki_slices, ctx->gemm_ws, ctx->gemm_ws_bytes, ctx->cs, fa, fb), "Ozaki GEMM");
    *nl += 6;   // (memset + colmax + 2 splits, or cached leaf forms made once) + GEMM (+ split-K reduce)
    return;
  }
  ZgemmProblem p = problem_for(n.op, g.Lt, g.N, g.S, a, b, out);
  ck(launch_zgemm(p, ctx->gemm_ws, ctx->gemm_ws_bytes, ctx->num_sms, ctx->cs, nl), "contraction kernel");
}

// Issues the plan on the three streams.  Returns the number of kernel launches.
int issue(cc_ctx* ctx, bool time_kernels, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* kev,
          std::vector<int>* kev_kind) {
  NvtxRange nv("cc issue_opbyop");
  const Dag& g = *ctx->dag;
  const int64_t per_t_m = 16LL * g.N * g.N;
  cudaStream_t st[3] = {ctx->cs, ctx->hs, ctx->ds};
  int nl = 0;
  ck(cudaEventRecord(ctx->ev_start, ctx->cs), "event");
  ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_start, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->ds, ctx->ev_start, 0), "wait");
  // consecutive TR_MM contractions share one batched trace launch; the batch is launched
  // before any other op is issued, and its source events right after
  int tr_kind = CC_TR_MM;                 // kind of the pending batch
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
    ck(launch_trace_batch(ta.data(), tb.data(), tout.data(), int(tops.size()), g.Lt, trace_shape(tr_kind, g.N, g.S),
                          ctx->trace_ws, ctx->cs),
       "contract-all batch");
    ++nl;
    if (time_kernels) {
      ck(cudaEventRecord(e1, ctx->cs), "event");
      kev->push_back({e0, e1});
      kev_kind->push_back(tr_kind);
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
    if (op.kind == OP_CONTRACT && is_root_kind(g.nodes[size_t(op.node)].op)) {
      const Node& n = g.nodes[size_t(op.node)];
      if (!tops.empty() && n.op != tr_kind) flush_tr();   // a batch holds one shape
      tr_kind = n.op;
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
    for (int32_t d : op.deps) ck(cudaStreamWaitEvent(s, ctx->events[size_t(d)], 0), "wait");
    for (const Move& m : op.pre_moves) {      // compaction (physical plan): non-overlapping D2D moves
      ck(cudaMemcpyAsync(ctx->arena + m.dst, ctx->arena + m.src, size_t(m.bytes), cudaMemcpyDeviceToDevice, s), "move");
      ctx->run_moves += m.bytes;
    }
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
        ctx->count_copy(true, op.bytes);
        break;
      }
      case OP_P2P_IN: {
        // from the peer tier (stashed tensor) or the leaf's peer home copy (E-10, E-11)
        const void* src = op.peer_off >= 0 ? static_cast<const void*>(ctx->peer_tier + op.peer_off)
                                           : peer_leaf_src(ctx, op.node);
        ck(cudaMemcpyAsync(ctx->arena + op.dev_off, src, size_t(op.bytes), cudaMemcpyDefault, s), "P2P in");
        ctx->count_op_copy(OP_P2P_IN, op.bytes);
        break;
      }
      case OP_P2P_OUT:
        ck(cudaMemcpyAsync(ctx->peer_tier + op.peer_off, ctx->arena + op.dev_off, size_t(op.bytes), cudaMemcpyDefault, s),
           "P2P out");
        ctx->count_op_copy(OP_P2P_OUT, op.bytes);
        break;
      case OP_D2H:
        ctx->count_copy(false, op.bytes);
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
    if (is_root_kind(n.op) != (cls == 1)) continue;
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
        if (is_root_kind(n.op) != (cls == 1)) continue;
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

}  // namespace ccx
