// C ABI (include/cc.h).  Argument checks, ordering (CC_E_STATE) and error mapping; the
// work happens in the exec/ and host/ translation units.
#include "internal.hpp"

#include <mutex>

static thread_local std::string g_err = "no error";   // context-free calls (ctx == NULL)

static cc_status fail(cc_ctx* ctx, const Error& e) {
  if (ctx) ctx->err = e.what();
  else g_err = e.what();
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


namespace {
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

const char* cc_last_error(const cc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

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
  ctx->n_time_parts = 1;
  rebuild_dag(ctx);
  API_END
}

cc_status cc_partition_grid(cc_ctx* ctx, int32_t n_tree_parts, int32_t n_time_parts, int32_t part) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  if (n_tree_parts < 1 || n_time_parts < 1 || part < 0 || int64_t(part) >= int64_t(n_tree_parts) * n_time_parts)
    throw Error(CC_E_INVAL, "bad grid partition");
  // a degenerate grid is a plain TIME (one tree part) or TREES (one time part) split
  ctx->n_parts = n_tree_parts == 1 ? n_time_parts : n_tree_parts;
  ctx->n_time_parts = n_tree_parts == 1 ? 1 : n_time_parts;
  ctx->part = part;
  ctx->mode = n_tree_parts == 1 ? 0 : (n_time_parts == 1 ? 1 : 2);
  rebuild_dag(ctx);
  API_END
}

cc_status cc_part_info(cc_ctx* ctx, cc_part_stats* out) {
  if (!ctx || !out) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  Dag full(ctx->input);
  std::vector<int32_t> owner;
  const bool trees = ctx->n_parts > 1 && ctx->mode != 0;
  std::vector<int32_t> parts = trees ? tree_parts(full, ctx->n_parts, nullptr, &owner) : std::vector<int32_t>();
  const int32_t pt = trees ? ctx->part / (ctx->mode == 2 ? ctx->n_time_parts : 1) : 0;
  const Dag& g = *ctx->dag;
  const int64_t lt = ctx->t1 - ctx->t0;
  cc_part_stats s{};
  s.n_trees = int64_t(g.trees.size());
  for (const Node& n : g.nodes) {
    bool mine = true;
    if (trees) {
      const int32_t u = full.idx(n.id);
      mine = owner[size_t(u)] >= 0 && parts[size_t(owner[size_t(u)])] == pt;
    }
    if (n.leaf()) {
      s.leaf_bytes += n.size;
      if (!mine) s.replicated_leaf_bytes += n.size;
    } else {
      const int64_t wu = contraction_weight(g, n, lt);
      ++s.n_contr;
      s.work += wu;
      if (!mine) s.replicated_work += wu;
    }
  }
  *out = s;
  API_END
}

cc_status cc_leaf_owners(cc_ctx* ctx, int64_t* leaf_ids, int32_t* owners, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  if (ctx->n_parts <= 1 || ctx->mode == 0) throw Error(CC_E_STATE, "leaf owners need a TREES or GRID partition");
  Dag full(ctx->input);
  std::vector<int32_t> owner;
  std::vector<int32_t> parts = tree_parts(full, ctx->n_parts, nullptr, &owner);
  int64_t n = 0;
  for (size_t u = 0; u < full.nodes.size(); ++u)
    if (full.nodes[u].leaf() && owner[u] >= 0) {
      if ((leaf_ids || owners) && n >= cap) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
      if (leaf_ids) leaf_ids[n] = full.nodes[u].id;
      if (owners) owners[n] = parts[size_t(owner[u])];
      ++n;
    }
  if (n_out) *n_out = n;
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
  NvtxRange nv("cc_schedule");
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
  if (cfg->peer_cap_bytes < 0 || cfg->n_peer_leaves < 0 || (cfg->n_peer_leaves > 0 && !cfg->peer_leaves))
    throw Error(CC_E_INVAL, "bad peer tier configuration");
  std::vector<uint8_t> peer_home(g.nodes.size(), 0);
  for (int64_t i = 0; i < cfg->n_peer_leaves; ++i) {
    auto it = g.index.find(cfg->peer_leaves[i]);
    if (it == g.index.end()) {
      bool other_part = false;   // a leaf of another TREES part: ignored
      for (const auto& nn : ctx->input.nodes) other_part |= nn.id == cfg->peer_leaves[i];
      if (!other_part) throw Error(CC_E_UNKNOWN_NODE, "unknown peer leaf " + std::to_string(cfg->peer_leaves[i]));
      continue;
    }
    if (!g.nodes[size_t(it->second)].leaf()) throw Error(CC_E_INVAL, "peer leaf " + std::to_string(cfg->peer_leaves[i]) + " is not a leaf");
    peer_home[size_t(it->second)] = 1;
  }
  ctx->lp = lru_plan(g, order, cfg->cap_bytes, (cfg->flags & CC_EVICT_NEXT_USE) ? EVICT_NEXT_USE : EVICT_LRU,
                     cfg->peer_cap_bytes, &peer_home);
  ctx->peer_home = std::move(peer_home);
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
  s.p2p_out_count = ctx->lp.p2p_out_count;
  s.p2p_out_bytes = ctx->lp.p2p_out_bytes;
  s.p2p_in_count = ctx->lp.p2p_in_count;
  s.p2p_in_bytes = ctx->lp.p2p_in_bytes;
  s.peer_peak_bytes = ctx->lp.peer_peak;
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

cc_status cc_phys_plan(cc_ctx* ctx, int64_t pool_bytes, int32_t compact, cc_phys_stats* out) {  // compact = flags
  if (!ctx || pool_bytes <= 0) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->scheduled) throw Error(CC_E_STATE, "no schedule");
  const Dag& g = *ctx->dag;
  std::vector<uint8_t> on_dev(g.nodes.size(), 0);
  for (size_t u = 0; u < g.nodes.size() && u < ctx->leaf_dev.size(); ++u) on_dev[u] = ctx->leaf_dev[u] != nullptr;
  PhysPlan pp = build_phys(g, ctx->lp, on_dev, pool_bytes, ALIGN, (compact & 2) ? RangeAlloc::NEXT_FIT : RangeAlloc::BEST_FIT,
                           ctx->peer_tier_bytes, false, (compact & 1) != 0);
  if (out) {
    *out = cc_phys_stats{};
    out->pool_high_water = pp.pool_high_water;
    out->n_moves = pp.n_moves;
    out->move_bytes = pp.move_bytes;
    out->host_pool_bytes = pp.host_pool_bytes;
  }
  ctx->phys_probe = std::move(pp);
  API_END
}

cc_status cc_scratch_of(cc_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->scheduled) throw Error(CC_E_STATE, "no schedule");
  *out = scratch_sizes(ctx).total;
  API_END
}

cc_status cc_phys_ops(cc_ctx* ctx, cc_phys_op* out, int64_t cap, int64_t* n_out) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  const auto& ops = ctx->phys_probe.ops;
  const Dag& g = *ctx->dag;
  int64_t n = 0;
  for (const auto& op : ops) n += 1 + int64_t(op.pre_moves.size());
  if (n_out) *n_out = n;
  if (out) {
    if (cap < n) throw Error(CC_E_BUFFER_TOO_SMALL, "buffer too small");
    int64_t k = 0;
    for (const auto& op : ops) {
      for (const auto& m : op.pre_moves)
        out[k++] = cc_phys_op{7, 0, g.nodes[size_t(m.node)].id, m.bytes, m.src, m.dst, -1, -1};
      const Node& nd = g.nodes[size_t(op.node)];
      out[k++] = cc_phys_op{op.kind, 0, nd.id, op.bytes, op.dev_off, -1, op.kind == OP_CONTRACT ? op.off_a : -1,
                            op.kind == OP_CONTRACT ? op.off_b : -1};
    }
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

cc_status cc_set_leaf_peer(cc_ctx* ctx, int64_t leaf_id, const void* dev, size_t bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!ctx->loaded) throw Error(CC_E_STATE, "no DAG loaded");
  const Dag& g = *ctx->dag;
  auto it = g.index.find(leaf_id);
  if (it == g.index.end()) {
    for (const auto& n : ctx->input.nodes)
      if (n.id == leaf_id) return CC_OK;   // a leaf of another TREES part
    throw Error(CC_E_UNKNOWN_NODE, "unknown leaf " + std::to_string(leaf_id));
  }
  const Node& n = g.nodes[size_t(it->second)];
  if (!n.leaf()) throw Error(CC_E_INVAL, "node " + std::to_string(leaf_id) + " is not a leaf");
  const int64_t full = tensor_bytes(n.op, ctx->input.dims.Lt, g.N, g.S);
  if (int64_t(bytes) != full) throw Error(CC_E_INVAL, "leaf " + std::to_string(leaf_id) + ": expected " + std::to_string(full) + " bytes");
  if (!dev) throw Error(CC_E_INVAL, "null peer pointer");
  ctx->leaf_peer[size_t(it->second)] = dev;
  ctx->release_graph();  // copy sources are baked into a captured graph
  API_END
}

// ---- CUDA IPC plumbing for the peer tier / leaf sharing between rank processes ----------
namespace {
std::mutex g_ipc_mu;
std::map<uintptr_t, void*> g_ipc_open;   // pointer handed out -> mapped base
}  // namespace

cc_status cc_ipc_export(const void* dev, uint8_t handle_out[64], uint64_t* offset_out) {
  cc_ctx* ctx = nullptr;
  if (!dev || !handle_out || !offset_out) return CC_E_INVAL;
  API_BEGIN
  using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static PFN_range range = nullptr;
  if (!range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      throw Error(CC_E_CUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_range>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev)) != CUDA_SUCCESS)
    throw Error(CC_E_INVAL, "cc_ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  ck(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle_out, &h, 64);
  *offset_out = uint64_t(reinterpret_cast<uintptr_t>(dev) - uintptr_t(base));
  API_END
}

cc_status cc_ipc_open(const uint8_t handle[64], uint64_t offset, void** dev_out) {
  cc_ctx* ctx = nullptr;
  if (!handle || !dev_out) return CC_E_INVAL;
  API_BEGIN
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* base = nullptr;
  ck(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  void* p = static_cast<char*>(base) + offset;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_open[reinterpret_cast<uintptr_t>(p)] = base;
  *dev_out = p;
  API_END
}

cc_status cc_ipc_close(void* dev) {
  cc_ctx* ctx = nullptr;
  API_BEGIN
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_open.find(reinterpret_cast<uintptr_t>(dev));
    if (it == g_ipc_open.end()) throw Error(CC_E_INVAL, "cc_ipc_close: not a pointer from cc_ipc_open");
    base = it->second;
    g_ipc_open.erase(it);
  }
  ck(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
  API_END
}

cc_status cc_set_peer_tier(cc_ctx* ctx, void* dev, size_t bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if ((dev == nullptr) != (bytes == 0)) throw Error(CC_E_INVAL, "peer tier: pointer and size must both be set or both be 0");
  ctx->peer_tier = static_cast<char*>(dev);
  ctx->peer_tier_bytes = int64_t(bytes);
  ctx->phys_valid = false;
  ctx->release_graph();
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
  if (flags & (2 | 4 | 8 | 32)) throw Error(CC_E_INVAL, "cc_execute_async: flags bits 1, 2, 3 and 5 need a blocking cc_execute");
  execute(ctx, flags, false, nullptr);
  API_END
}

cc_status cc_get_options(cc_ctx* ctx, cc_options* out) {
  if (!ctx || !out) return CC_E_INVAL;
  *out = ctx->opt;
  return CC_OK;
}

cc_status cc_set_options(cc_ctx* ctx, const cc_options* opt) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  if (!opt) throw Error(CC_E_INVAL, "null options");
  const cc_options& o = *opt;
  auto bit = [](int32_t v) { return v == 0 || v == 1; };
  if (!bit(o.trace_fusion) || !bit(o.copy_reorder) || !bit(o.early_copies) || !bit(o.precopy) ||
      !bit(o.ozaki_leaf_cache) || o.ozaki_slices < 4 || o.ozaki_slices > 7 || o.h2d_chunk_bytes < 0 ||
      !(o.tr_ratio >= 0.0 && o.tr_ratio <= 64.0) || o.debug < 0 || o.debug > 3 || !bit(o.slice_major) ||
      !bit(o.leaf_slots) || !bit(o.trace_groups))
    throw Error(CC_E_INVAL, "option out of range");
  ctx->opt = o;
  if (!ctx->host_only) ctx->release_phys();   // scratch sizes, graphs and dataflow metadata depend on them
  ctx->phys_valid = false;
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
  for (int k = 0; k < CC_N_OPS; ++k) {
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
static cc_status direct_trace(cc_ctx* ctx, int op, const void* A, const void* B, void* c, int32_t Lt, int32_t N,
                              int32_t S) {
  API_BEGIN
  ctx->need_device();
  if (!A || !B || !c || Lt <= 0 || N <= 0 || S <= 0) throw Error(CC_E_INVAL, "bad kernel arguments");
  const TraceShape sh = trace_shape(op, N, S);
  ensure_ws(ctx->direct_tr_ws, ctx->direct_tr_ws_bytes, trace_workspace_bytes(Lt, sh));
  // counters must be zero; a previous direct call with another Lt may have left partials there
  ck(cudaMemsetAsync(ctx->direct_tr_ws, 0, size_t(Lt) * 4 * 32, ctx->cs), "memset");
  ck(launch_trace(A, B, c, Lt, sh, ctx->direct_tr_ws, ctx->cs), "contract-all kernel");
  API_END
}

cc_status cc_tr_mm(cc_ctx* ctx, const void* A, const void* B, void* c, int32_t Lt, int32_t N) {
  if (!ctx) return CC_E_INVAL;
  return direct_trace(ctx, CC_TR_MM, A, B, c, Lt, N, 1);
}
cc_status cc_bb1(cc_ctx* ctx, const void* A, const void* B, void* T, int32_t Lt, int32_t N, int32_t S) {
  if (!ctx) return CC_E_INVAL;
  return direct_gemm(ctx, CC_BB1, A, B, T, Lt, N, S);
}
cc_status cc_bt2(cc_ctx* ctx, const void* A, const void* X, void* C, int32_t Lt, int32_t N, int32_t S) {
  if (!ctx) return CC_E_INVAL;
  return direct_gemm(ctx, CC_BT2, A, X, C, Lt, N, S);
}
cc_status cc_bb3(cc_ctx* ctx, const void* A, const void* B, void* c, int32_t Lt, int32_t N, int32_t S) {
  if (!ctx) return CC_E_INVAL;
  return direct_trace(ctx, CC_BB3, A, B, c, Lt, N, S);
}

size_t cc_gemm_ozaki_workspace_bytes(int32_t op, int32_t Lt, int32_t N, int32_t S, int32_t n_slices) {
  if (!is_gemm_kind(op) || Lt <= 0 || N <= 0 || S <= 0 || n_slices < 4 || n_slices > 7)
    return 0;
  return ozaki_workspace_bytes(problem_for(op, Lt, N, op == CC_MM1 ? 1 : S, nullptr, nullptr, nullptr), n_slices, Lt);
}

cc_status cc_gemm_ozaki(cc_ctx* ctx, int32_t op, const void* A, const void* B, void* C, int32_t Lt, int32_t N,
                        int32_t S, int32_t n_slices, void* workspace, size_t workspace_bytes) {
  if (!ctx) return CC_E_INVAL;
  API_BEGIN
  ctx->need_device();
  if (!is_gemm_kind(op) || !A || !B || !C || !workspace || Lt <= 0 || N <= 0 || S <= 0 ||
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
  for (int op : GEMM_OPS)
    ws = std::max(ws, zgemm_workspace_bytes(problem_for(op, Lt, N, S, nullptr, nullptr, nullptr), 148));
  size_t tws = 0;
  for (int op : TRACE_OPS) tws = std::max(tws, trace_workspace_bytes(Lt, trace_shape(op, N, S)));
  return ws + tws + size_t(Lt) * 16 * 3 * 65536 + (size_t(16) << 20);
}

}  // extern "C"
