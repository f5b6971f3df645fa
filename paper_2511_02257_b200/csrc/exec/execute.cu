// cc_execute's driver: engine choice, CUDA graphs, statistics.
#include "internal.hpp"

namespace ccx {

void execute(cc_ctx* ctx, int32_t flags, bool blocking, cc_exec_stats* stats) {
  NvtxRange nv("cc_execute");
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
  // dataflow executor only; opt.precopy = 0 disables).  Every pre-copied range lies inside the
  // pool the scratch layout leaves (and the capped physical limit), so a stray copy can never
  // land in scratch or outside the arena; if preparation fails, the compute stream is ordered
  // after the stray copies before the error returns.
  ctx->pre_n = 0;
  ctx->run_h2d = ctx->run_d2h = ctx->run_p2p_in = ctx->run_p2p_out = ctx->run_moves = 0;
  std::vector<int64_t> pre_off;
  if (ctx->opt.precopy && ctx->opt.early_copies && ctx->opt.h2d_chunk_bytes == 0 && !ctx->phys_valid &&
      !ctx->dag->abstract && !(flags & (2 | 4 | 8 | 16 | 64 | 128))) {
    const Dag& g0 = *ctx->dag;
    int64_t limit = (ctx->arena_bytes - scratch_sizes(ctx).total) / ALIGN * ALIGN;
    if (ctx->cap > 0) limit = std::min(limit, round_up(ctx->cap + ctx->cap / 4, ALIGN));
    int64_t off = 0;
    for (size_t j = 0; j < ctx->lp.ops.size() && j < 4; ++j) {
      const auto& lop = ctx->lp.ops[j];
      if (lop.kind != OP_H2D) break;
      const int32_t u = lop.node;
      const Node& n0 = g0.nodes[size_t(u)];
      if (!n0.leaf() || ctx->leaf_dev[size_t(u)] || !ctx->leaf_host[size_t(u)]) break;
      if (off + round_up(n0.size, ALIGN) > limit) break;
      if (!ctx->ev_precopy) ck(cudaEventCreateWithFlags(&ctx->ev_precopy, cudaEventDisableTiming), "event");
      if (j == 0) {
        ck(cudaEventRecord(ctx->ev_precopy, ctx->cs), "event");   // after all earlier work on cs
        ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_precopy, 0), "wait");
      }
      const int64_t per_t_m = 16LL * g0.N * g0.N;
      const int64_t per_t = n0.op == CC_LEAF_M ? per_t_m : per_t_m * g0.S * g0.N;
      const char* src = static_cast<const char*>(ctx->leaf_host[size_t(u)]) + int64_t(ctx->t0) * per_t;
      ck(cudaMemcpyAsync(ctx->arena + off, src, size_t(n0.size), cudaMemcpyHostToDevice, ctx->hs), "H2D");
      ctx->count_copy(true, n0.size);
      pre_off.push_back(off);
      off += round_up(n0.size, ALIGN);
    }
    if (!pre_off.empty()) {
      ck(cudaEventRecord(ctx->ev_precopy, ctx->hs), "event");
      ctx->pre_n = int(pre_off.size());
    }
  }
  try {
    prepare_phys(ctx);
  } catch (...) {
    if (ctx->pre_n > 0) cudaStreamWaitEvent(ctx->cs, ctx->ev_precopy, 0);
    ctx->pre_n = 0;
    throw;
  }
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
    // (profiles/r02_configs_final.txt): GEMMs with N >= 512 (c5 N = 512 part 0.74 vs
    // 0.91 s, N = 1024 part 1.84 vs 3.35 s; at N = 256 the worker wins, 1.21 vs 1.41 s), or
    // baryon GEMMs with N >= 128 (c4 1.41 vs 1.57 s)
    const Dag& gd = *ctx->dag;
    bool gemm = false, baryon = false;
    for (const auto& n : gd.nodes) {
      gemm |= is_gemm_kind(n.op);
      baryon |= is_gemm_kind(n.op) && n.op != CC_MM1;
    }
    if (gemm && (gd.N >= 512 || (baryon && gd.N >= 128))) flags |= 64;
    flags &= ~128;
  }
  ctx->mm1_ozaki = (flags & 64) != 0;
  if (ctx->mm1_ozaki) oz_cache_reset(ctx);
  if (flags & 12) {
    kernel_only(ctx, (flags & 4) ? 0 : 1, stats);
    return;
  }
  const bool use_graph = (flags & 1) != 0;
  // a plan with compaction moves runs op by op (the moves are copies on the allocating op's stream)
  const bool legacy = (flags & 16) != 0 || (flags & 2) != 0 || (flags & 64) != 0 || ctx->pp.n_moves > 0;
  const bool time_kernels = (flags & 2) != 0 && !use_graph;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;
  std::vector<int> kev_kind;
  if (!legacy) {
    prepare_dataflow(ctx, ctx->opt.early_copies != 0);
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
      ctx->graph_h2d = ctx->run_h2d;     // the copies the graph carries
      ctx->graph_d2h = ctx->run_d2h;
      ctx->graph_p2p_in = ctx->run_p2p_in;
      ctx->graph_p2p_out = ctx->run_p2p_out;
      ctx->graph_moves = ctx->run_moves;
    } else {
      ctx->run_h2d = ctx->graph_h2d;
      ctx->run_d2h = ctx->graph_d2h;
      ctx->run_p2p_in = ctx->graph_p2p_in;
      ctx->run_p2p_out = ctx->graph_p2p_out;
      ctx->run_moves = ctx->graph_moves;
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
    stats->h2d_bytes = ctx->run_h2d;      // counted as enqueued (the plan's: cc_plan_stats)
    stats->d2h_bytes = ctx->run_d2h;
    stats->p2p_in_bytes = ctx->run_p2p_in;
    stats->p2p_out_bytes = ctx->run_p2p_out;
    stats->move_bytes = ctx->run_moves;
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
    for (int k = 0; k < CC_N_OPS; ++k) ks += ctx->ktimes.seconds[k];
    stats->kernel_seconds = ks;
  }
  cudaEventDestroy(t_begin);
  cudaEventDestroy(t_end);
}

}  // namespace ccx
