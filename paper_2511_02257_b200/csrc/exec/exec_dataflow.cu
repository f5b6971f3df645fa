// Dataflow execution: the plan's contractions as work items of the persistent worker
// (kernels/dataflow.hpp), copies on the copy streams, synchronised through integer slots.
#include "internal.hpp"

namespace ccx {
namespace {

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
  if (op.kind == OP_P2P_IN)   // peer tier (E-10) or a peer-homed leaf (E-11)
    return {op.peer_off >= 0 ? static_cast<const void*>(ctx->peer_tier + op.peer_off) : peer_leaf_src(ctx, op.node),
            ctx->arena + op.dev_off};
  if (op.kind == OP_P2P_OUT) return {ctx->arena + op.dev_off, ctx->peer_tier + op.peer_off};
  return {ctx->arena + op.dev_off, ctx->host_pool + op.host_off};
}
cudaMemcpyKind copy_kind(int32_t op_kind) {
  return op_kind == OP_H2D ? cudaMemcpyHostToDevice : op_kind == OP_D2H ? cudaMemcpyDeviceToHost : cudaMemcpyDefault;
}

// One plan copy on `s`: C time-slice chunks, each followed by a flag write (value = chunks
// done) — the dataflow worker's items wait on the flag (chunk of their slice, kernels/dataflow.hpp).
void enqueue_copy(cc_ctx* ctx, cudaStream_t s, const void* src, void* dst, size_t bytes, int32_t op_kind,
                  int32_t chunks, int32_t flag_slot) {
  const cudaMemcpyKind kind = copy_kind(op_kind);
  const Dag& g = *ctx->dag;
  const size_t per_t = bytes / size_t(std::max<int64_t>(g.Lt, 1));
  for (int32_t ch = 0; ch < chunks; ++ch) {
    // chunk ch: slices [ch*Lt/C, (ch+1)*Lt/C)
    const size_t t0 = chunks == 1 ? 0 : size_t(int64_t(ch) * g.Lt / chunks);
    const size_t t1 = chunks == 1 ? 0 : size_t(int64_t(ch + 1) * g.Lt / chunks);
    const size_t off = t0 * per_t, len = chunks == 1 ? bytes : (t1 - t0) * per_t;
    // a device-to-device copy (peer tier, peer-homed leaf, kind Default) may run as a copy
    // kernel, which could never start while the persistent worker holds every SM: the worker
    // leaves one SM free when the plan has peer copies (issue_dataflow)
    ck(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len, kind, s), "copy");
    ctx->count_op_copy(op_kind, int64_t(len));
    if (df_write_fn()(s, reinterpret_cast<CUdeviceptr>(ctx->df_sync + flag_slot), cuuint32_t(ch + 1), 0) != CUDA_SUCCESS)
      throw Error(CC_E_CUDA, "cuStreamWriteValue32 failed");
  }
}

}  // namespace

// early: start the wait-free H2D copies at the head of the copy order on the H2D stream as
// soon as that order is known, so they overlap the rest of the host-side preparation (queues,
// tensor maps, upload); the next issue_dataflow only adds their flag writes.
void prepare_dataflow(cc_ctx* ctx, bool early) {
  if (ctx->df_valid) return;
  NvtxRange nv("cc prepare_dataflow");
  if (ctx->opt.debug & 1) fprintf(stderr, "[cc] prepare_dataflow\n");
  prepare_phys(ctx);
  PhaseTimer tmr("prepare_dataflow", (ctx->opt.debug & 2) != 0);
  const Dag& g = *ctx->dag;
  const auto& ops = ctx->pp.ops;
  const int64_t Lt = g.Lt, N = g.N;
  const int32_t n_ops = int32_t(ops.size());
  const int64_t per_t_m = 16LL * g.N * g.N;
  // sync slots (done counters of compute ops, flags of copies) and H2D chunk counts
  std::vector<int32_t> slot(size_t(n_ops), -1), target(size_t(n_ops), 0), df_index(size_t(n_ops), -1);
  int32_t n_sync = 0;
  // per-time-slice done counters of GEMMs (every op is batched over time slices, reading V-1):
  // a trace or GEMM reading slice t of a GEMM's output waits only for that slice's tiles
  std::vector<int32_t> slice_slot(size_t(n_ops), -1), items_per_slice(size_t(n_ops), 0);
  // opt.h2d_chunk_bytes: H2D copies in time-slice chunks of about that size (default off: every
  // chunk costs a stream memory operation, measured ~8 us of copy-engine idle each on B200)
  const int64_t h2d_chunk = ctx->opt.h2d_chunk_bytes > 0 ? std::max<int64_t>(4096, ctx->opt.h2d_chunk_bytes) : INT64_MAX;
  for (int32_t i = 0; i < n_ops; ++i) {
    const PhysOp& op = ops[size_t(i)];
    if (op.stream == S_NONE) continue;
    slot[size_t(i)] = n_sync++;
    if (op.kind == OP_CONTRACT && Lt > 1 && is_gemm_kind(g.nodes[size_t(op.node)].op)) {
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
  // 0b. early H2D copies.  A leaf H2D whose device range no earlier op of the plan touched
  // (fresh pool memory, e.g. every leaf slot) waits on nothing and nothing earlier depends on it:
  // it may be issued first, before the dependency analysis, so the copy engine starts while
  // the host builds the rest.  These copies are ordered greedily by the work they enable:
  // next = the leaf that completes the leaf set (closure in the DAG) of the most estimated
  // compute time, so the GEMMs — most of the step — start early and little is left once the
  // last leaf lands.  Option copy_reorder = 0 keeps plan order.
  std::vector<int32_t> early_seq;
  std::vector<uint8_t> is_early(size_t(n_ops), 0);
  int32_t n_first = 0;                                 // early copies already enqueued (plan ops 0..n-1)
  {
    // byte ranges of the pool touched so far in plan order (merged intervals start -> end)
    std::map<int64_t, int64_t> touched;
    auto touch = [&](int64_t off, int64_t bytes) {
      if (off < 0) return;
      int64_t lo = off, hi = off + bytes;
      auto it = touched.upper_bound(lo);
      if (it != touched.begin() && std::prev(it)->second >= lo) --it;
      while (it != touched.end() && it->first <= hi) {
        lo = std::min(lo, it->first);
        hi = std::max(hi, it->second);
        it = touched.erase(it);
      }
      touched[lo] = hi;
    };
    auto fresh = [&](int64_t off, int64_t bytes) {
      auto it = touched.upper_bound(off);
      if (it != touched.end() && it->first < off + bytes) return false;
      return it == touched.begin() || std::prev(it)->second <= off;
    };
    for (int32_t i = 0; i < n_ops; ++i) {
      const PhysOp& op = ops[size_t(i)];
      const Node& n = g.nodes[size_t(op.node)];
      const int64_t rb = round_up(n.size, ALIGN);
      if (op.kind == OP_H2D && op.stream == S_H2D && n.leaf() && fresh(op.dev_off, rb)) {
        is_early[size_t(i)] = 1;
        early_seq.push_back(i);
      }
      if (op.kind == OP_H2D || op.kind == OP_D2H || op.kind == OP_P2P_IN || op.kind == OP_P2P_OUT) touch(op.dev_off, rb);
      if (op.kind == OP_CONTRACT) {
        if (op.loc_a == LOC_POOL) touch(op.off_a, round_up(g.nodes[size_t(n.l)].size, ALIGN));
        if (op.loc_b == LOC_POOL) touch(op.off_b, round_up(g.nodes[size_t(n.r)].size, ALIGN));
        touch(op.dev_off, rb);
      }
    }
    const int reorder = ctx->opt.copy_reorder;
    // the plan's first leaf copies start now, before the ordering of the others is computed
    // (they head the order either way); the first pre_n of them were even started by
    // execute() before the physical plan existed, and only get their flag writes here
    if (early && !early_seq.empty()) {
      // zero the sync area on the compute stream (after all earlier work there); the H2D
      // stream's flag writes and copies follow it (and the previous replay's readers)
      ck(cudaMemsetAsync(ctx->df_sync_base, 0, sz_sync, ctx->cs), "memset");
      ck(cudaEventRecord(ctx->ev_pre, ctx->cs), "event");
      ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_pre, 0), "wait");
      int pre = ctx->pre_n;
      for (int j = 0; j < pre; ++j)
        if (size_t(j) >= early_seq.size() || early_seq[size_t(j)] != j || target[size_t(j)] != 1) pre = 0;
      if (pre == 0 && ctx->pre_n > 0) ck(cudaStreamWaitEvent(ctx->cs, ctx->ev_precopy, 0), "wait");
      for (int j = 0; j < pre; ++j)   // hs order: pre-copies, (wait for the zeroing), flags
        if (df_write_fn()(ctx->hs, reinterpret_cast<CUdeviceptr>(ctx->df_sync + slot[size_t(j)]), 1u, 0) != CUDA_SUCCESS)
          throw Error(CC_E_CUDA, "cuStreamWriteValue32 failed");
      if (pre == 0) {
        const int32_t i = early_seq[0];
        const auto ep = copy_endpoints(ctx, ops[size_t(i)]);
        enqueue_copy(ctx, ctx->hs, ep.first, ep.second, size_t(ops[size_t(i)].bytes), OP_H2D,
                     target[size_t(i)] < 0 ? -target[size_t(i)] : 1, slot[size_t(i)]);
        n_first = 1;
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
  }
  // early copies: the rest of the wait-free copies, each followed by its flag write, so they
  // overlap the rest of the host-side preparation (the sync area was zeroed on the compute
  // stream above, which does not wait for any copy: the worker polls the flags).
  ctx->df_early.assign(size_t(n_ops), 0);
  ctx->df_early_active = false;
  if (early && !early_seq.empty()) {
    size_t q_issued = 0;
    for (int32_t i : early_seq) {
      const PhysOp& op = ops[size_t(i)];
      ctx->df_early[size_t(i)] = 1;
      if (q_issued++ < size_t(n_first)) continue;     // enqueued before the ordering
      const auto ep = copy_endpoints(ctx, op);
      enqueue_copy(ctx, ctx->hs, ep.first, ep.second, size_t(op.bytes),
                   OP_H2D, target[size_t(i)] < 0 ? -target[size_t(i)] : 1, slot[size_t(i)]);
    }
    ctx->df_early_active = true;
  }
  tmr.lap("early copies");
  // 1. data dependencies over the device pool and the host pool
  RWTracker dev(ctx->pool_bytes), host(std::max<int64_t>(ctx->pp.host_pool_bytes, 1)),
      peer(std::max<int64_t>(ctx->peer_tier_bytes, 1));
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
    } else if (op.kind == OP_P2P_IN && op.stream != S_NONE) {
      dev.write(op.dev_off, rb, i, d);
      if (op.peer_off >= 0) peer.read(op.peer_off, rb, i, d);
    } else if (op.kind == OP_P2P_OUT && op.stream != S_NONE) {
      dev.read(op.dev_off, rb, i, d);
      peer.write(op.peer_off, rb, i, d);
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
    const bool fuse = ctx->opt.trace_fusion != 0 && df_supports_fusion();
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
    if (is_root_kind(n.op)) {
      const TraceShape sh = trace_shape(n.op, N, g.S);
      const int64_t P = df_trace_pieces(sh);
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
      d.tr_G = sh.G;
      d.tr_Gj = n.op == CC_BB3 ? sh.Gj : 0;
      d.tr_S = n.op == CC_BB3 ? int32_t(g.S) : 1;
      // partial slots (P > 1) come from a ring assigned in queue order below
      d.tmap = int32_t(tmaps.size() / 256);
      tmaps.resize(tmaps.size() + 256);
      const bool ok = n.op == CC_BB3 ? df_encode_bb3_maps(tmaps.data() + size_t(d.tmap) * 256, a, b, Lt, N, g.S)
                                     : df_encode_trace_maps(tmaps.data() + size_t(d.tmap) * 256, a, b, Lt, N, &d.tr_cw);
      if (!ok) throw Error(CC_E_CUDA, "TMA descriptor encoding failed");
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
  std::vector<int32_t> tr_run(size_t(n_ops), -1);         // trace run of each TR op (3a', 3b)
  std::vector<int64_t> avail(size_t(n_ops), 0);
  // 3. queue order: a topological order of the plan's ops (compute and copy; consecutive
  // copies on one stream are chained, since a copy stream runs in plan order) that delays each
  // TR_MM op by DF_TR_DELAY compute positions, so a trace item is usually claimed after its
  // operand GEMMs completed (no worker blocks on it) while the GEMMs behind it keep the DMMA
  // pipes busy.  Any topological order keeps the dataflow deadlock-free (dataflow.hpp).
  {
    constexpr int64_t delay = 8;
    std::vector<std::vector<int32_t>> succ(static_cast<size_t>(n_ops));
    std::vector<int32_t> indeg(static_cast<size_t>(n_ops), 0), rank(static_cast<size_t>(n_ops), 0);
    std::vector<int32_t> chain_prev(size_t(n_ops), -1);   // previous copy on the same stream (issue order)
    for (int st : {int(S_H2D), int(S_D2H)})
      for (size_t k = 1; k < copy_seq[st].size(); ++k) chain_prev[size_t(copy_seq[st][k])] = copy_seq[st][k - 1];
    // avail: the H2D issue position after which an op's inputs can all be there
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
      const bool tr = op.kind == OP_CONTRACT && is_root_kind(g.nodes[size_t(op.node)].op);
      return avail[size_t(i)] * (int64_t(n_ops) + delay + 1) + int64_t(rank[size_t(i)]) + (tr ? delay : 0);
    };
    std::priority_queue<std::pair<int64_t, int32_t>, std::vector<std::pair<int64_t, int32_t>>, std::greater<>> ready;
    for (int32_t i = 0; i < n_ops; ++i)
      if (slot[size_t(i)] >= 0 && indeg[size_t(i)] == 0) ready.push({key(i), i});
    std::vector<int32_t> order;
    // pop segment of each op: it changes at every op that is not a trace (GEMMs AND copies), so
    // traces with equal segments were popped back to back (3a')
    std::vector<int32_t> pop_seg(size_t(n_ops), -1);
    int32_t seg = 0;
    while (!ready.empty()) {
      const int32_t i = ready.top().second;
      ready.pop();
      const bool trace = ops[size_t(i)].kind == OP_CONTRACT && is_root_kind(g.nodes[size_t(ops[size_t(i)].node)].op);
      if (!trace) ++seg;
      pop_seg[size_t(i)] = seg;
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
    // 3a'. trace runs (option trace_groups): TR ops popped back to back by the topological sort
    // (no GEMM and no copy between them: equal pop segment) are mutually independent with the
    // same predecessors and successors, so any permutation of a run keeps the merged order —
    // copies included, the deadlock-freedom witness (dataflow.hpp) — topological.  Each run is
    // clustered by shared operand (greedy: the operand most traces of the run read first), so
    // traces reading the same tensor are adjacent in the TR queue and — interleaved slice by
    // slice below — read its time slices from L2 after the first.
    if (ctx->opt.trace_groups) {
      auto is_tr = [&](int32_t i) { return df_index[size_t(i)] >= 0 && gops[size_t(df_index[size_t(i)])].kind == 1; };
      int32_t runs = 0;
      for (size_t k = 0; k < order.size();) {
        if (!is_tr(order[k])) {
          ++k;
          continue;
        }
        size_t e = k;
        while (e < order.size() && is_tr(order[e]) && pop_seg[size_t(order[e])] == pop_seg[size_t(order[k])]) ++e;
        if (e - k > 1) {
          std::vector<int32_t> rest(order.begin() + int64_t(k), order.begin() + int64_t(e)), out;
          auto opnd = [&](int32_t i, int w) {
            const DfOp& d = gops[size_t(df_index[size_t(i)])];
            return w ? d.B : d.A;
          };
          for (int32_t x : cluster_by_operand(rest.size(), [&](size_t x, int w) { return opnd(rest[x], w); }))
            out.push_back(rest[size_t(x)]);
          std::copy(out.begin(), out.end(), order.begin() + int64_t(k));
        }
        for (size_t x = k; x < e; ++x) tr_run[size_t(order[x])] = runs;
        ++runs;
        k = e;
      }
    }
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
  // 3b. item order within each queue.  Op-major (an op's items contiguous, in queue order),
  // or — option slice_major — time slice by time slice within each run of ops whose inputs
  // become available at the same copy position (avail): all ops' items of slice 0, then of
  // slice 1, ..., so the GEMM outputs of a slice are traced while still in L2 and a leaf
  // slice is read by every GEMM using it back to back.  Requires every dependency between
  // contractions to be a per-slice RAW on an operand (no memory-reuse or ring dependencies)
  // and no fused traces; the merged order (segment by segment, slice by slice, GEMM items
  // before trace items, ops in queue order) stays topological, so the dataflow stays
  // deadlock-free (dataflow.hpp).
  std::vector<int32_t> gitem_op, gitem_local, titem_op, titem_local;
  {
    auto ips_of = [&](int32_t i, const DfOp& d) -> int64_t {
      return d.kind == 1 ? int64_t(d.P) : int64_t(items_per_slice[size_t(i)]);
    };
    bool sm = ctx->opt.slice_major != 0 && Lt > 1 && fusedv.empty();
    for (int32_t i = 0; sm && i < n_ops; ++i) {
      const PhysOp& op = ops[size_t(i)];
      if (op.kind != OP_CONTRACT || slot[size_t(i)] < 0) continue;
      if (!ring_deps[size_t(i)].empty()) sm = false;
      if (df_index[size_t(i)] >= 0 && !is_root_kind(g.nodes[size_t(op.node)].op) && items_per_slice[size_t(i)] <= 0)
        sm = false;
      for (int32_t j : deps[size_t(i)]) {
        if (ops[size_t(j)].kind != OP_CONTRACT) continue;
        const bool raw = j == wr_a[size_t(i)] || j == wr_b[size_t(i)];
        if (!raw || items_per_slice[size_t(j)] <= 0) sm = false;
      }
    }
    auto build = [&](const std::vector<DfOp>& v, const std::vector<int32_t>& plan, std::vector<int32_t>& iop,
                     std::vector<int32_t>& iloc) {
      for (size_t k0 = 0; k0 < v.size();) {
        size_t k1 = k0 + 1;
        if (sm)
          while (k1 < v.size() && avail[size_t(plan[k1])] == avail[size_t(plan[k0])]) ++k1;
        const bool trq = !v.empty() && v[0].kind == 1;
        if (!sm && trq && tr_run[size_t(plan[k0])] >= 0) {
          // a trace run in op-major mode: chunks of consecutive TR ops that never share a
          // partial-ring slot (< DF_TRACE_RING ops) go time slice by time slice, so the
          // clustered traces read a shared operand's slice from L2 after the first
          k1 = k0 + 1;
          while (k1 < v.size() && k1 - k0 < size_t(DF_TRACE_RING) && tr_run[size_t(plan[k1])] == tr_run[size_t(plan[k0])])
            ++k1;
          for (int64_t t = 0; t < Lt; ++t)
            for (size_t k = k0; k < k1; ++k)
              for (int64_t x = t * v[k].P; x < (t + 1) * v[k].P; ++x) {
                iop.push_back(int32_t(k));
                iloc.push_back(int32_t(x));
              }
        } else if (!sm) {
          for (int32_t x = 0; x < v[k0].n_items; ++x) {
            iop.push_back(int32_t(k0));
            iloc.push_back(x);
          }
        } else {
          for (int64_t t = 0; t < Lt; ++t)
            for (size_t k = k0; k < k1; ++k) {
              const int64_t ips = ips_of(plan[k], v[k]);
              for (int64_t x = t * ips; x < (t + 1) * ips; ++x) {
                iop.push_back(int32_t(k));
                iloc.push_back(int32_t(x));
              }
            }
        }
        k0 = k1;
      }
    };
    build(gops, gplan, gitem_op, gitem_local);
    build(tops, tplan, titem_op, titem_local);
    if (int64_t(gitem_op.size()) != g_items || int64_t(titem_op.size()) != t_items)
      throw Error(CC_E_STATE, "dataflow: item order lost items");
    ctx->df_slice_major = sm;
    if (gitem_op.empty()) { gitem_op.push_back(0); gitem_local.push_back(0); }
    if (titem_op.empty()) { titem_op.push_back(0); titem_local.push_back(0); }
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
        // a trace, or a GEMM batched over the same time slices, reading slice t of this GEMM's
        // output (RAW on an operand; reuse deps stay whole-op) waits for that slice only
        const bool raw = j == wr_a[size_t(i)] || j == wr_b[size_t(i)];
        if (items_per_slice[size_t(j)] > 0 && (traces || (raw && items_per_slice[size_t(i)] > 0))) {
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
  const size_t sz_gi = round_up(int64_t(gitem_op.size() * 4), 256), sz_ti = round_up(int64_t(titem_op.size() * 4), 256);
  const size_t sz_f = round_up(int64_t(std::max<size_t>(fusedv.size(), 1) * sizeof(DfFused)), 256);
  const size_t total = sz_g + sz_t + 2 * sz_d + sz_m + 2 * sz_gi + 2 * sz_ti + sz_f;
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
  char* pgl = pti + sz_ti;
  char* ptl = pgl + sz_gi;
  char* pf = ptl + sz_ti;
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
    put(pgl, gitem_local.data(), gitem_local.size() * 4);
    put(ptl, titem_local.data(), titem_local.size() * 4);
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
  da.q = DfQueue{reinterpret_cast<const DfOp*>(pg), reinterpret_cast<const int32_t*>(pgi),
                 reinterpret_cast<const int32_t*>(pgl), int32_t(gops.size()),
                 g_items, heads};
  da.qt = DfQueue{reinterpret_cast<const DfOp*>(pt), reinterpret_cast<const int32_t*>(pti),
                  reinterpret_cast<const int32_t*>(ptl), int32_t(tops.size()),
                  t_items, heads + 1};
  {
    da.Lt = int32_t(Lt);
    da.ahead_g = 2;   // items a CTA's scheduler holds claimed-but-unpublished per queue
    da.ahead_t = 2;
  }
  ctx->df_gemm_items = g_items;
  ctx->df_trace_items = t_items;
  da.prof = nullptr;
  da.prof_t = nullptr;
  tmr.lap("upload");
  ctx->df_valid = true;
}

static int32_t ops_kind_of(cc_ctx* ctx, int32_t op) { return ctx->pp.ops[size_t(op)].kind; }

// Enqueues one dataflow replay; returns the number of kernel launches.
int issue_dataflow(cc_ctx* ctx, bool time_copies) {
  NvtxRange nv("cc issue_dataflow");
  const Dag& g = *ctx->dag;
  int nl = 0;
  const bool dbg = (ctx->opt.debug & 1) != 0;
#define DBG(...) do { if (dbg) { fprintf(stderr, "[cc] " __VA_ARGS__); fputc('\n', stderr); fflush(stderr); } } while (0)
  PhaseTimer tmr("issue_dataflow", (ctx->opt.debug & 2) != 0);
  DBG("issue_dataflow: %zu copies, %lld gemm items, %lld trace items", ctx->df_copies.size(),
      (long long)ctx->df_gemm_items, (long long)ctx->df_trace_items);
  if (!ctx->df_early_active) ck(cudaMemsetAsync(ctx->df_sync_base, 0, ctx->df_sync_bytes, ctx->cs), "memset");
  ck(cudaEventRecord(ctx->ev_start, ctx->cs), "event");
  ck(cudaStreamWaitEvent(ctx->hs, ctx->ev_start, 0), "wait");
  ck(cudaStreamWaitEvent(ctx->ds, ctx->ev_start, 0), "wait");
  // The worker goes first: copy streams may block on stream memory ops waiting for its
  // counters, and a driver can stall the host's enqueue of further memory ops until the
  // device makes progress — so the kernel they wait for must already be queued.
  if (ctx->df_gemm_items + ctx->df_trace_items > 0) {
    // one SM stays free when the plan has peer (device-to-device) copies (see enqueue_copy)
    const bool p2p = ctx->pp.p2p_in_bytes > 0 || ctx->pp.p2p_out_bytes > 0;
    ck(df_launch(ctx->df_gemm, ctx->num_sms - (p2p ? 1 : 0), ctx->cs), "dataflow worker");
    DBG("worker launched");
    ++nl;
    if (ctx->df_n_fused > 0) {
      ck(df_launch_fused_finish(ctx->df_gemm.fused, ctx->df_n_fused, g.Lt, ctx->cs), "fused trace finish");
      ++nl;
    }
  }
  cudaStream_t st[3] = {ctx->cs, ctx->hs, ctx->ds};
  for (const int32_t kk : ctx->df_issue) {
    const size_t k = size_t(kk);
    const auto& c = ctx->df_copies[k];
    cudaStream_t s = st[c.stream];
    for (int32_t e : c.wait_events) ck(cudaStreamWaitEvent(s, ctx->df_events[size_t(e)], 0), "wait");
    for (const auto& wv : c.wait_values)
      if (df_wait_fn()(s, reinterpret_cast<CUdeviceptr>(ctx->df_sync + wv.first), cuuint32_t(wv.second),
                       CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        throw Error(CC_E_CUDA, "cuStreamWaitValue32 failed");
    DBG("copy %zu: stream %d bytes %zu waits %zu/%zu", k, c.stream, c.bytes, c.wait_values.size(), c.wait_events.size());
    // copies started during preparation (flags included) are skipped
    if (!(ctx->df_early_active && ctx->df_early[size_t(c.op)]))
      enqueue_copy(ctx, s, c.src, c.dst, c.bytes, ops_kind_of(ctx, c.op), c.chunks, c.flag_slot);
    DBG("copy %zu enqueued", k);
    if (c.source) ck(cudaEventRecord(ctx->df_events[k], s), "event");
  }
  DBG("copies enqueued");
  ctx->df_early_active = false;   // later replays copy everything and zero the sync area on cs
  if (time_copies) {
    ck(cudaEventRecord(ctx->ev_copy_h, ctx->hs), "event");
    ck(cudaEventRecord(ctx->ev_copy_d, ctx->ds), "event");
  }
  ctx->copy_timed = time_copies;
  tmr.lap("copies");
  DBG("workers launched");
  tmr.lap("worker");
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

}  // namespace ccx
