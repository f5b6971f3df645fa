/*
 * cc.h — C ABI of the correlator-contraction engine (libcc.so).
 *
 * The engine executes the binary, batched, complex-double tensor contractions of a
 * Redstar-style contraction DAG (§II-B) in a memory-minimising
 * sequential schedule (§II-C problem statement, l.248; sibling scheduler §III-A,
 * tree scheduler §III-B), releasing intermediates at last use (l.62, l.207-211) and
 * evicting least-recently-used tensors to pinned host memory when the device pool is
 * full (MemHC, l.136-139; eviction definition l.913).  "P:n" below = PAPER.md line n.
 *
 * Conventions
 *  - Every function returns cc_status (0 = CC_OK, < 0 = error); no C++ exception crosses
 *    the ABI.  cc_last_error(ctx) gives a message for the last failing call on ctx
 *    (cc_last_error(NULL): the calling thread's last failing context-free call).
 *  - complex128 tensors are interleaved (re, im) doubles, row-major, time slice t
 *    outermost: meson node [Lt][N][N], baryon node [Lt][S][N][N][N] (S = spin
 *    components, 64 in P:59), root value [Lt].  Byte sizes 16*Lt*N^2, 16*Lt*S*N^3, 16*Lt.
 *  - Node ids and tree ids are caller-chosen int64, unique; ties in the schedulers are
 *    broken by ascending id (readings S-1, S-3, T-1).
 *  - A cc_ctx is one device (or host-only when device < 0); not thread-safe.
 *  - Ordering: cc_create -> cc_load_dag -> [cc_partition] -> cc_schedule ->
 *    cc_set_leaf* -> cc_execute -> cc_correlator / cc_root_value.  Calls out of order
 *    return CC_E_STATE.  cc_schedule / cc_execute may be repeated (same plan re-run).
 */
#ifndef CC_H
#define CC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CC_OK = 0,
  CC_E_INVAL = -1,            /* bad argument                                         */
  CC_E_PARSE = -2,            /* text format error (message carries the line number)  */
  CC_E_CYCLE = -3,            /* the operand relation has a cycle                     */
  CC_E_INCONSISTENT = -4,     /* duplicate id, operand kinds do not fit the op, ...   */
  CC_E_MULTIROOT = -5,        /* a root shared by two trees / a parentless non-root   */
  CC_E_UNKNOWN_NODE = -6,     /* operand / root / tree id not declared                */
  CC_E_NOT_CLOSED = -7,       /* reserved (trees are closures of their roots)         */
  CC_E_INFEASIBLE = -8,       /* operands + output of one contraction exceed cap      */
  CC_E_STATE = -9,            /* call out of order, or op not allowed on this ctx     */
  CC_E_BUFFER_TOO_SMALL = -10,
  CC_E_CUDA = -11,            /* CUDA runtime error (message has the CUDA string)     */
  CC_E_NOMEM = -12            /* arena / host allocation failed                       */
} cc_status;

/* Node kinds.  Index semantics (readings V-1 and T4-1..T4-4; P:120, P:806-813,
 * P:867):
 *   CC_MM1   (meson A, meson B)   C[t,i,k]       = sum_j A[t,i,j] B[t,j,k]          O(N^3)
 *   CC_BM1   (baryon A, meson M)  C[t,s,i,j,l]   = sum_k A[t,s,i,j,k] M[t,k,l]      O(N^4)
 *   CC_BB2   (baryon A, baryon B) C[t,i,l]       = sum_s sum_{j,k} A[t,s,i,j,k] B[t,s,j,k,l]
 *   CC_TR_MM (meson A, meson B)   c[t]           = sum_{i,j} A[t,i,j] B[t,j,i]   (root only:
 *                                  "contract all")
 *   BxBxB (tritium class, Table II P:813 O(N^5); sizes O(N^2)/O(N^3)/O(N^4)):
 *   CC_BB1   (baryon A, baryon B) T[t,i,j,l,m]   = sum_s sum_k A[t,s,i,j,k] B[t,s,k,l,m]
 *                                  -> tetraquark node [Lt][N][N][N][N], O(S N^5)
 *   CC_BT2   (baryon A, tetra X)  C[t,s,m,i,j]   = sum_{k,l} A[t,s,m,k,l] X[t,k,l,i,j]
 *                                  -> baryon node, O(S N^5)
 *   CC_BB3   (baryon A, baryon B) c[t]           = sum_s sum_{i,j,k} A[t,s,i,j,k] B[t,s,k,j,i]
 *                                  (root only: baryon x baryon "contract all", O(S N^3))
 * CC_LEAF_X / CC_OP_X are abstract nodes of explicit size for scheduling-only DAGs
 * (e.g. Table I); a DAG containing them can be scheduled/planned, not executed. */
typedef enum {
  CC_LEAF_M = 0, CC_LEAF_B = 1, CC_MM1 = 2, CC_BM1 = 3, CC_BB2 = 4, CC_TR_MM = 5,
  CC_LEAF_X = 6, CC_OP_X = 7, CC_BB1 = 8, CC_BT2 = 9, CC_BB3 = 10
} cc_op;
#define CC_N_OPS 11

typedef struct { int32_t Lt, N, S; } cc_dims;

/* a, b: ordered operand ids (left, right), -1 for leaves.  size: 0 = derive
 * from the kind and dims; > 0 = explicit bytes (required for abstract nodes; must match
 * the derived size for typed nodes). */
typedef struct { int64_t id; int32_t op; int32_t pad_; int64_t a, b; int64_t size; } cc_node;
/* A tree is its root plus the closure of the root under operands. */
typedef struct { int64_t tree_id; int64_t root; } cc_tree;
/* Correlator term: C_corr[t] += (re + i im) * root_tree[t]. */
typedef struct { int64_t corr_id; int64_t tree_id; double re, im; } cc_term;

/* CC_RSGS: RS-GS-like baseline — Redstar's similarity sort of trees (the paper's
 * RS-GS comparison of §IV) under DESIGN.md readings R-1..R-4. */
typedef enum { CC_SIBLING = 0, CC_TREE = 1, CC_GIVEN = 2, CC_RSGS = 3 } cc_algo;

/* cc_sched_cfg.flags bit 0: evict by next use instead of LRU (reading E-9; the
 * whole schedule is known offline, so the victim is the resident non-operand whose next read
 * is farthest away, ties to the least recently used). */
#define CC_EVICT_NEXT_USE 1

typedef struct {
  int32_t algo;               /* cc_algo                                                   */
  int32_t flags;              /* CC_EVICT_NEXT_USE or 0 (LRU)                              */
  uint64_t seed;              /* reserved (reading S-1 pins the "random leaf" to lowest id) */
  int64_t cap_bytes;          /* device pool capacity for the LRU plan; <= 0: unbounded     */
  const int64_t* given_order; /* CC_GIVEN: contraction order (node ids), n_given entries    */
  int64_t n_given;
  /* Peer-HBM tier (readings E-10, E-11; NVLink instead of the PCIe
   * bus the paper names as the bottleneck).  peer_cap_bytes > 0: a victim
   * with no off-device copy (an intermediate's first eviction, or a leaf) is copied to a peer
   * GPU's HBM while that many bytes remain, and re-fetched from there; the copy lives until
   * release.  peer_leaves: ids of leaves whose home copy is in a peer GPU's HBM (cross-GPU
   * leaf sharing: every fetch of them is a peer copy, never H2D).  0 / NULL: no peer tier. */
  int64_t peer_cap_bytes;
  const int64_t* peer_leaves;
  int64_t n_peer_leaves;
} cc_sched_cfg;

/* Logical plan statistics (integers are bit-exact with the oracle).
 * peak / transient_peak: device bytes after releases / right after producing an output
 * (§II-C M_i and reading G-5); evictions / h2d / d2h: readings E-1..E-5. */
typedef struct {
  int64_t n_contr, peak, transient_peak, evictions, h2d_count, d2h_count,
          h2d_bytes, d2h_bytes, host_peak_bytes, model_peak, model_transient_peak;
  double sched_seconds;       /* scheduler wall time only (Table IV analogue) */
  double plan_seconds;        /* LRU plan + physical placement                              */
  int64_t arena_high_water;   /* physical pool bytes used (>= peak; fragmentation headroom)  */
  int64_t p2p_out_count, p2p_out_bytes, p2p_in_count, p2p_in_bytes, peer_peak_bytes;
                              /* peer-tier copies (E-10, E-11): evictions copied to the peer
                                 tier, fetches from a peer; bytes in the peer tier at most  */
} cc_plan_stats;

typedef struct {
  double seconds;             /* cc_execute time: device events from entry (before any plan
                                 preparation) to the last op; time to solution            */
  double kernel_seconds;      /* sum of contraction-kernel durations (0 unless profiled)    */
  double flops;               /* algorithmic flops: MM1 8LtN^3, BM1/BB2 8LtSN^4, TR 8LtN^2   */
  double hbm_bytes;           /* algorithmic HBM bytes of the kernels                       */
  int64_t h2d_bytes, d2h_bytes; /* bytes copied, counted as the executor enqueues each copy (a
                                   dropped or duplicated copy shows here; the plan's own counts
                                   are cc_plan_stats; device-resident leaves: 0).  Includes the
                                   up to 4 early leaf copies a first dataflow execute starts
                                   before its physical plan exists, when that plan then places
                                   them elsewhere or runs op by op (compaction)            */
  int64_t n_kernels;          /* kernel launches issued by this execute                     */
  double copy_seconds;        /* start -> last H2D/D2H copy done (blocking stream-mode
                                 dataflow execute with copies; else 0)                     */
  int64_t p2p_in_bytes, p2p_out_bytes; /* peer-tier copies, counted as enqueued             */
  int64_t move_bytes;         /* compaction device-to-device moves (physical plan), enqueued  */
  int64_t pad_;
} cc_exec_stats;

/* One op of the physical plan (cc_plan_ops). kind: 0 H2D, 1 D2H (evict with copy),
 * 2 DROP (evict, no copy), 3 CONTRACT, 4 FREE (release at last use), 5 P2P_OUT (evict with a
 * copy to the peer tier), 6 P2P_IN (fetch from a peer GPU's HBM). */
typedef struct { int32_t kind; int32_t pad_; int64_t node; int64_t bytes; int64_t offset; } cc_plan_op;

typedef struct cc_ctx cc_ctx;

/* device < 0: host-only context (load/validate/schedule/plan only).
 * dev_arena/arena_bytes: caller-owned device memory the pool sub-allocates (may be NULL/0
 *   on a host-only ctx).  The top `CC_SCRATCH` bytes of it are kernel workspace (split-K
 *   partials; outside the logical capacity, reading E-7).
 * streams: caller-owned cudaStream_t (NULL: the library creates its own). */
cc_status cc_create(cc_ctx** out, int device, void* dev_arena, size_t arena_bytes,
                    void* compute_stream, void* h2d_stream, void* d2h_stream);
void cc_destroy(cc_ctx* ctx);
const char* cc_last_error(const cc_ctx* ctx);
const char* cc_version(void);

/* Copies the inputs; builds G=(V,E), validates, computes ranks (Eq. 1) and F_v/F_e. */
cc_status cc_load_dag(cc_ctx* ctx, const cc_dims* dims, const cc_node* nodes, int64_t n_nodes,
                      const cc_tree* trees, int64_t n_trees, const cc_term* terms, int64_t n_terms);
/* Text format, one record per line, '#' comments:
 *   dims <Lt> <N> <S>
 *   node <id> leafM|leafB|leafX [size <bytes>]
 *   node <id> MM1|BM1|BB2|TR_MM|OPX <a> <b> [size <bytes>]
 *   tree <tree_id> <root>
 *   term <corr_id> <tree_id> <re> <im>                                               */
cc_status cc_load_dag_file(cc_ctx* ctx, const char* path);

typedef struct { int64_t V, E, k, n_contr, n_leaves, max_rank, n_corr; double F_v, F_e; } cc_dag_stats;
cc_status cc_dag_info(cc_ctx* ctx, cc_dag_stats* out);

/* Restrict the context to one part of an n_parts split:
 * mode 0 TIME: time slices [part*Lt/n, (part+1)*Lt/n) of every tensor (no replication);
 * mode 1 TREES: a contiguous, flop-balanced chunk of the trees in tree-scheduler
 *   selection order, with the sub-DAG they need (shared nodes replicated).
 * Call after cc_load_dag, before cc_schedule.  n_parts == 1 restores the full DAG.  Errors:
 * CC_E_INVAL for part outside [0, n_parts), an unknown mode, or a TIME part that owns no time
 * slice (n_parts > Lt), CC_E_STATE before cc_load_dag. */
cc_status cc_partition(cc_ctx* ctx, int32_t n_parts, int32_t part, int32_t mode);
/* GRID split (reading M-2): n_tree_parts TREES parts x n_time_parts TIME parts; part
 * p in [0, n_tree_parts * n_time_parts) is TREES part p / n_time_parts restricted to the time
 * slices of TIME part p % n_time_parts (e.g. c5 at N = 1024 over 8 GPUs: the per-GPU plan of a
 * TIME-only split does not fit HBM).  Errors as cc_partition. */
cc_status cc_partition_grid(cc_ctx* ctx, int32_t n_tree_parts, int32_t n_time_parts, int32_t part);
/* Work of the current part (reading M-3; replicas "counted as overhead and
 * reported"): work = sum of flops/8 of its contractions at its slice count (MM1 Lt N^3, ...,
 * abstract: 1 each); replicated_* = the share of nodes whose owner (the part of the first
 * selected tree containing them) is another part.  No partition: replicated = 0. */
typedef struct { int64_t n_trees, n_contr, work, replicated_work, leaf_bytes, replicated_leaf_bytes; } cc_part_stats;
cc_status cc_part_info(cc_ctx* ctx, cc_part_stats* out);
/* Owner part of every leaf of the full DAG under the current TREES / GRID split (reading
 * E-11: the rank that loads a shared leaf over PCIe; the others read its copy over NVLink
 * with cc_set_leaf_peer).  leaf_ids / owners may be NULL (count query).  CC_E_STATE without a
 * TREES / GRID partition. */
cc_status cc_leaf_owners(cc_ctx* ctx, int64_t* leaf_ids, int32_t* owners, int64_t cap, int64_t* n_out);
/* Trees of the current part (ids, ascending); n_out receives the count. */
cc_status cc_part_trees(cc_ctx* ctx, int64_t* out, int64_t cap, int64_t* n_out);
/* Time-slice range [t0, t1) of the loaded part (the whole [0, Lt) unless a TIME partition is
 * active): where this part's correlator slices go in the full [n_corr][Lt] buffer. */
cc_status cc_part_time_range(cc_ctx* ctx, int32_t* t0, int32_t* t1);

/* Runs the scheduler (Alg. 1-3 or Alg. 4-8), then the LRU plan at cfg->cap_bytes and the
 * physical placement in the arena.  order_out (may be NULL: size query) receives the
 * contraction order; n_order its length.  stats may be NULL. */
cc_status cc_schedule(cc_ctx* ctx, const cc_sched_cfg* cfg, int64_t* order_out, int64_t order_cap,
                      int64_t* n_order, cc_plan_stats* stats);
/* §II-C trace of the current schedule: M_0..M_n (n+1 entries) and transient_1..n. */
cc_status cc_memory_trace(cc_ctx* ctx, int64_t* m_out, int64_t* transient_out, int64_t cap, int64_t* n_out);
/* The op queue of the current plan, in order. */
cc_status cc_plan_ops(cc_ctx* ctx, cc_plan_op* out, int64_t cap, int64_t* n_out);
/* Tree order of the last CC_TREE (selection order) or CC_RSGS (similarity chain) schedule (tree ids). */
cc_status cc_tree_order(cc_ctx* ctx, int64_t* out, int64_t cap, int64_t* n_out);
/* Host-side placement query (no device needed): the physical plan of the current schedule over a
 * pool of pool_bytes.  flags bit 0: an allocation that finds no free block clears a window by
 * device-to-device moves of small resident tensors (what cc_execute falls back to when next fit
 * and best fit both fail; such plans execute op by op); bit 1: next fit instead of best fit.
 * CC_E_NOMEM if it does not fit. */
typedef struct { int64_t pool_high_water, n_moves, move_bytes, host_pool_bytes; } cc_phys_stats;
cc_status cc_phys_plan(cc_ctx* ctx, int64_t pool_bytes, int32_t flags, cc_phys_stats* out);
/* The ops of the last cc_phys_plan, compaction moves inline before the op that needs them:
 * kind as cc_plan_op, 7 = MOVE (offset = source, dst = destination); offset = the op's pool
 * offset (copy target / output), off_a / off_b = a contraction's operand offsets (-1 for a
 * caller device leaf or when not a contraction). */
typedef struct { int32_t kind; int32_t pad_; int64_t node; int64_t bytes; int64_t offset, dst, off_a, off_b; } cc_phys_op;
cc_status cc_phys_ops(cc_ctx* ctx, cc_phys_op* out, int64_t cap, int64_t* n_out);
/* Exact bytes cc_execute reserves at the top of the arena for kernel workspace and tables with
 * the current DAG and options (the pool is the rest, rounded down to 1 KiB). */
cc_status cc_scratch_of(cc_ctx* ctx, int64_t* out);
/* Per-step op queue as CSV (step, op, node, bytes, offset, device_used). */
cc_status cc_plan_dump(cc_ctx* ctx, const char* csv_path);

/* Leaf data.  host: caller-owned pinned (or registered) host buffer of the full leaf
 * ([Lt_full,...], all time slices; a TIME part reads its own slices), valid until the
 * last cc_execute returns.  dev: caller-owned device buffer of the leaf restricted to the
 * current part (inputs already resident in HBM: no H2D is issued for it; evicting it is
 * a no-op).  bytes must equal the (full / part) leaf size. */
cc_status cc_set_leaf(cc_ctx* ctx, int64_t leaf_id, const void* host, size_t bytes);
cc_status cc_set_leaf_device(cc_ctx* ctx, int64_t leaf_id, const void* dev, size_t bytes);
/* Peer-homed leaf (E-11): dev is the address, in this process, of the full leaf ([Lt_full,...])
 * in a peer GPU's HBM (a CUDA IPC mapping of the owner rank's buffer, or any device pointer
 * cudaMemcpyAsync(cudaMemcpyDefault) can read — a buffer on this GPU works the same way),
 * caller-owned, valid and holding the data until the last cc_execute returns.  Required
 * for every leaf named in cc_sched_cfg.peer_leaves; each P2P_IN copies the part's slices. */
cc_status cc_set_leaf_peer(cc_ctx* ctx, int64_t leaf_id, const void* dev, size_t bytes);
/* The peer-HBM eviction tier region (E-10): caller-owned device memory (normally a CUDA IPC
 * mapping of a peer GPU's buffer; any device pointer works), at least the plan's
 * peer_peak_bytes plus fragmentation.  P2P_OUT copies are placed in it best-fit; cc_execute
 * fails with CC_E_NOMEM if they do not fit, CC_E_STATE if the plan has peer copies and no
 * region is set.  dev NULL / bytes 0 removes it. */
cc_status cc_set_peer_tier(cc_ctx* ctx, void* dev, size_t bytes);
/* CUDA IPC plumbing between the one-process-per-GPU ranks (peer tier, leaf sharing):
 * cc_ipc_export: a 64-byte handle of the device allocation holding dev (any address inside a
 *   cudaMalloc'ed block, e.g. a torch tensor) and dev's offset in it; CC_E_INVAL if dev is not
 *   device memory.
 * cc_ipc_open: maps another process's handle (same GPU or a peer GPU), returns base + offset;
 *   the mapping stays until cc_ipc_close(that pointer).  Context-free; thread-safe. */
cc_status cc_ipc_export(const void* dev, uint8_t handle_out[64], uint64_t* offset_out);
cc_status cc_ipc_open(const uint8_t handle[64], uint64_t offset, void** dev_out);
cc_status cc_ipc_close(void* dev);

/* Replays the plan on the device: H2D / D2H on the copy streams, contractions on the
 * compute stream, event dependencies for RAW on data and WAR on reused memory; blocking.
 * flags bit 0: capture/replay as a CUDA graph; bit 1: time every kernel (kernel_seconds; not
 * with bit 0).  bit 2 / bit 3: kernel-only replay of the plan's GEMM-kind (MM1/BM1/BB2) /
 * TR_MM launches alone, in plan order, as a cached graph, after a full execute: stats->seconds
 * = device time of the replay, n_kernels = launches, flops/hbm_bytes = their algorithmic work
 * (average launch duration for the roofline, without host launch overhead).  The default
 * executor is the dataflow one (persistent DMMA-tile and trace workers, kernels/dataflow.hpp);
 * bit 4 selects op-by-op launches instead; bit 5 records the per-item timeline
 * (cc_dataflow_profile); bit 6 runs every MM1 / BM1 / BB2 on the tcgen05 INT8 Ozaki engine
 * (cc_gemm_ozaki, 5 slices; leaves split once per execute; implies op-by-op launches); bit 7
 * (CC_EXEC_AUTO) chooses bit 6 or the dataflow worker by the measured rule of DESIGN §7 (the
 * Ozaki engine for GEMMs with N >= 512, or baryon GEMMs with N >= 128). */
#define CC_EXEC_OZAKI 64
#define CC_EXEC_AUTO 128
cc_status cc_execute(cc_ctx* ctx, int32_t flags, cc_exec_stats* stats);
/* Enqueue-only variant (no host sync): work is ordered on the compute stream.  Takes the same
 * flags as cc_execute except bits 1 (per-kernel timing), 2 / 3 (kernel-only replays) and 5
 * (profiling), which need a host sync: CC_E_INVAL. */
cc_status cc_execute_async(cc_ctx* ctx, int32_t flags);

/* Executor options of one context (defaults in brackets; cc_get_options returns the current
 * values).  They change how the plan is executed, never what it computes: results are
 * bit-identical across copy_reorder / early_copies / precopy / h2d_chunk_bytes /
 * ozaki_leaf_cache, and equal within V-4's tolerance across trace_fusion (a fused trace sums
 * in tile order).  Setting options drops cached graphs and dataflow metadata.
 *   trace_fusion      dataflow: compute a TR_MM inside the GEMM producing its later operand [0]
 *   copy_reorder      dataflow: order wait-free leaf H2D copies by the work they enable [1]
 *   early_copies      dataflow: start wait-free leaf copies while the metadata is built [1]
 *   precopy           dataflow: start up to 4 leading leaf copies before the physical plan [1]
 *   ozaki_leaf_cache  Ozaki engine: split every leaf once per execute [1]
 *   ozaki_slices      Ozaki engine: INT8 slices per operand, 4..7 [5]
 *   h2d_chunk_bytes   dataflow: H2D copies in time-slice chunks of about this size, each with its
 *                     own completion flag; 0: whole tensors [0]
 *   tr_ratio          ignored (the dataflow worker's traces run in their own warps since round 2;
 *                     the field keeps the struct layout) [0]
 *   debug             bit 0: executor trace on stderr; bit 1: host phase timings on stderr [0]
 *   slice_major       dataflow: order the work items time slice by time slice within each group
 *                     of ops whose inputs arrive together, so a slice's GEMM outputs are traced
 *                     (and its leaves reused) while they are still in L2; applies when every
 *                     dependency between contractions is per time slice [1]
 *   leaf_slots        unbounded plans: place every host leaf in a fixed slot of the pool so no
 *                     leaf copy waits for freed memory (falls back when the pool cannot hold the
 *                     leaves next to the plan's intermediates) [1]
 *   trace_groups      dataflow: traces adjacent in the queue (no other work between them) are
 *                     clustered by shared operand, and (op-major queues) run in chunks time
 *                     slice by time slice, so a shared operand's slices are read from L2 after
 *                     the first [1]
 * Errors: CC_E_INVAL for out-of-range values. */
typedef struct {
  int32_t trace_fusion, copy_reorder, early_copies, precopy, ozaki_leaf_cache, ozaki_slices;
  int64_t h2d_chunk_bytes;
  double tr_ratio;
  int32_t debug, slice_major;
  int32_t leaf_slots, trace_groups;
} cc_options;
cc_status cc_get_options(cc_ctx* ctx, cc_options* out);
cc_status cc_set_options(cc_ctx* ctx, const cc_options* opt);

/* Per-kind contraction-kernel time of the last cc_execute with flags bit 1 (kernels timed
 * with CUDA events on the compute stream): seconds[op], counts[op] for op = cc_op (CC_N_OPS each). */
cc_status cc_kernel_times(cc_ctx* ctx, double* seconds, int64_t* counts);

/* Progress of the dataflow executor (diagnostics; readable while a replay runs): out[0], out[1]
 * = items taken from the GEMM / TR queues, out[2..] = the sync slots (done counters of the
 * plan's contractions and copy-completion flags, in plan order). */
cc_status cc_dataflow_state(cc_ctx* ctx, int64_t* out, int64_t cap, int64_t* n_out);

/* Per-item timeline of the last cc_execute with flags bit 5 (dataflow profiling): for every
 * work item (GEMM queue first, then TR queue) 8 uint64: claim, dependencies-ready and
 * published times (%globaltimer, ns), the SM id, first-operand-arrival and end-of-stage-loop
 * times, the kind (0 GEMM, 1 TR_MM) and the first-arrival time again; then one record per
 * worker CTA (16 uint64): consumer cycles (clock64) waiting for GEMM / TR_MM stage data,
 * cycles in GEMM / TR_MM stage math and epilogues, GEMM / TR_MM stages consumed, SM id, GEMM
 * epilogue cycles, 8 reserved words.  out may be NULL (size query: 8*(n_gemm+n_trace+2*num_sms)). */
cc_status cc_dataflow_profile(cc_ctx* ctx, uint64_t* out, int64_t cap, int64_t* n_gemm, int64_t* n_trace);

/* Results.  out: 2*Lt_part doubles (interleaved complex) for the current part. */
cc_status cc_correlator(cc_ctx* ctx, int64_t corr_id, double* out, int32_t Lt);
cc_status cc_root_value(cc_ctx* ctx, int64_t tree_id, double* out, int32_t Lt);
/* Device buffer [n_corr][Lt_part] complex128 of all correlators (corr ids ascending), for
 * a torch / NCCL all-reduce; corr_ids (may be NULL) receives the ids in buffer order. */
cc_status cc_correlator_device_ptr(cc_ctx* ctx, void** dev_ptr, int64_t* n_corr, int64_t* corr_ids);
/* All correlators of the current part, [n_corr][Lt_part] interleaved complex (corr ids
 * ascending, as cc_correlator_device_ptr), into host memory `out` (cap doubles) with one copy
 * ordered after the last execute; pinned `out` makes it a DMA. */
cc_status cc_correlators(cc_ctx* ctx, double* out, int64_t cap);

/* Kernel entry points (the contraction kernels alone; used by the element-wise parity
 * tests and the roofline measurement).  All pointers are device pointers in the layouts
 * above; they run on the ctx compute stream and do not synchronise. */
cc_status cc_mm1(cc_ctx* ctx, const void* A, const void* B, void* C, int32_t Lt, int32_t N);
cc_status cc_bm1(cc_ctx* ctx, const void* A, const void* M, void* C, int32_t Lt, int32_t N, int32_t S);
cc_status cc_bb2(cc_ctx* ctx, const void* A, const void* B, void* C, int32_t Lt, int32_t N, int32_t S);
cc_status cc_tr_mm(cc_ctx* ctx, const void* A, const void* B, void* c, int32_t Lt, int32_t N);
/* BxBxB kinds alone (FP64 DMMA; layouts of the CC_BB1 / CC_BT2 / CC_BB3 definitions above):
 * A, B baryon [Lt][S][N][N][N]; T tetra [Lt][N][N][N][N]; C baryon; c [Lt]. */
cc_status cc_bb1(cc_ctx* ctx, const void* A, const void* B, void* T, int32_t Lt, int32_t N, int32_t S);
cc_status cc_bt2(cc_ctx* ctx, const void* A, const void* X, void* C, int32_t Lt, int32_t N, int32_t S);
cc_status cc_bb3(cc_ctx* ctx, const void* A, const void* B, void* c, int32_t Lt, int32_t N, int32_t S);
/* MM1 on the tcgen05 INT8 tensor cores by Ozaki splitting (DESIGN reading
 * V-6).  Same operation and layouts as cc_mm1 (C[t,i,k] = sum_j A[t,i,j] B[t,j,k], complex128
 * interleaved, [Lt][N][N], device pointers).  Each operand is scaled per row (A) / column (B)
 * by a power of two and split into n_slices (4..7) signed INT8 slices (balanced base-256
 * digits of a fixed-point value with 6 + 8 (n_slices - 1) fractional bits); the pairs (i, j)
 * with i + j <= n_slices - 1 are multiplied exactly (INT32 accumulation in TMEM) and summed in
 * FP64: |C - AB| <~ n_slices 2^(2 - 8 n_slices) 2N max_j|A[i,:]| max_k|B[:,k]| worst case,
 * ~sqrt(2N) times less typically (zero-mean digits).  workspace: caller-owned device memory of
 * cc_mm1_ozaki_workspace_bytes(Lt, N, n_slices) bytes (0 = invalid arguments).  Runs on the
 * ctx compute stream, does not synchronise.  Errors: CC_E_INVAL (bad sizes / null pointers,
 * N > 8192: INT32 accumulator bound), CC_E_BUFFER_TOO_SMALL, CC_E_CUDA. */
size_t cc_mm1_ozaki_workspace_bytes(int32_t Lt, int32_t N, int32_t n_slices);
cc_status cc_mm1_ozaki(cc_ctx* ctx, const void* A, const void* B, void* C, int32_t Lt, int32_t N, int32_t n_slices,
                       void* workspace, size_t workspace_bytes);
/* Any of the three contraction kinds on the Ozaki engine: op = CC_MM1 / CC_BM1 / CC_BB2 with
 * the layouts of cc_mm1 / cc_bm1 / cc_bb2 (S ignored for MM1).  BM1 splits the baryon's rows
 * (M = S N^2); BB2 contracts K = S N^2 in chunks of 8192 complex terms (INT32 bound), whose
 * FP64 partials are summed in chunk order (deterministic).  Time slices are processed in
 * batches that fit `workspace` (at least cc_gemm_ozaki_workspace_bytes(op, 1, N, S, s) bytes;
 * the full-batch size is returned for Lt).  Errors as cc_mm1_ozaki. */
size_t cc_gemm_ozaki_workspace_bytes(int32_t op, int32_t Lt, int32_t N, int32_t S, int32_t n_slices);
cc_status cc_gemm_ozaki(cc_ctx* ctx, int32_t op, const void* A, const void* B, void* C, int32_t Lt, int32_t N,
                        int32_t S, int32_t n_slices, void* workspace, size_t workspace_bytes);
/* The INT8 tcgen05 GEMM alone (pins the UMMA descriptors bit-exactly in the tests):
 * C[m][n] = sum_k A[m][k] B[n][k]; A int8 [M][K], B int8 [Nn][K] row-major, C int32 [M][Nn];
 * M % 128 == 0, Nn % 192 == 0 (a multiple of the tile width, 64 or 96 by build), K % 64 == 0,
 * K <= 2^17 (no INT32 overflow). */
cc_status cc_i8gemm_tn(cc_ctx* ctx, const int8_t* A, const int8_t* B, int32_t* C, int32_t M, int32_t Nn, int32_t K);
/* Synthetic leaf values (input generation, not the method; same recipe as synth/rng.py):
 * n complex elements starting at flat element e0 of leaf `leaf_id`, written to dev. */
cc_status cc_fill_synthetic(cc_ctx* ctx, void* dev, int64_t n, uint64_t seed, int64_t leaf_id,
                            int64_t e0, int32_t mode, double sigma);
/* Bytes of kernel workspace the ctx reserves at the top of the arena (plus, for DAGs with MM1
 * ops, the Ozaki leaf-form cache of execute flags bit 6 when it needs at most 1/8 of the arena). */
size_t cc_scratch_bytes(int32_t Lt, int32_t N, int32_t S);

#ifdef __cplusplus
}
#endif
#endif /* CC_H */
