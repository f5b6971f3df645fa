// Dataflow execution of a whole plan by a persistent worker kernel (host/device shared PODs).
//
// The plan's contractions become work items of two queues, each in one topological order of
// the plan: GEMM tiles (MM1/BM1/BB2; a tile may be split into k-chunks) and TR_MM block-pair
// ranges.  The worker is persistent (one CTA per SM); its producer holds at most one claimed
// item of each queue (atomic queue heads) and polls, without blocking, the integer sync slots
// of the items' op dependencies: done counters of earlier ops (RAW on operands, WAR/WAW on
// reused pool memory) and completion flags written by the copy streams after a copy
// (cuStreamWriteValue32).  Only stages of ready items enter the TMA ring.
// Deadlock freedom: let X be the earliest unfinished item in the merged topological order.
// Its dependencies are finished.  If X is claimed, its holder's producer sees it ready and
// issues it; every stage already in a ring belongs to a ready item, so the consumers drain
// the ring.  If X is unclaimed, every claimed item of X's queue precedes X and is therefore
// finished, so the next claim from that queue (which a producer makes as soon as it holds
// no item of that kind) is X.  Either way X finishes.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace cc {

struct DfOp {
  int32_t kind;           // 0 GEMM, 1 TRACE
  int32_t n_items;
  int64_t first_item;     // queue position of the op's first item (informational)
  int32_t sync_id;        // done counter (sync[sync_id] reaches n_items)
  int32_t slice_sync;     // GEMM with a [Lt, ...] output: per-time-slice done counters
                          // sync[slice_sync + t] (-1: none), so a trace of slice t waits only
                          // for that slice's tiles
  int32_t dep_begin, dep_count;
  // GEMM: C[b][m][n] = sum_k A[b][m][k] B[b][k][n] (zgemm semantics, kernels.hpp)
  int32_t tmap;           // tensor maps 2*tmap (A) and 2*tmap+1 (B)
  int32_t tiles_m, tiles_n, kt_per_o, KT, n_chunks;
  int64_t M, Nn, ldc, sCb;
  void* C;
  void* part;             // chunked: partial tiles [tile][chunk][slot]
  int* tile_cnt;          // chunked: per-tile finished-chunk counters (reset by the finisher)
  // TRACE: out[t] = sum_g sum_{i,j} A_g[t,i,j] B_g[t,j,i] over G sub-matrices per slice:
  // TR_MM G = 1; BB3 (reading T4-3) G = S N, g = (s, j) (kernels.hpp TraceShape)
  const void* A;
  const void* B;
  void* out;
  int64_t N, Lt;
  int32_t nb, P;          // 32x32 blocks per row; items (pieces) per time slice
  int32_t tr_G, tr_Gj;    // sub-matrices per slice; BB3: j extent (0 for TR_MM: 3-dim maps)
  int32_t tr_S;           // BB3: spin components (time-spin index of the maps: t S + s)
  int32_t tr_cw;          // TR_MM: chunk-wide maps (N % 8 == 0): one TMA box per 32x32 block
                          // (16 doubles x 32 rows x 4 column chunks) instead of four
  void* tr_part;          // [Lt][P] complex partials
  int* tr_cnt;            // [Lt] tickets (reset by the finisher)
  // GEMM with fused traces: after its k-tiles every output tile also computes, for each
  // fused TR_MM op f, sum over the tile of C[i][j] * X_f[j][i] (X_f = the trace's other
  // operand, two extra 32 KB stages per f), written per warp to fused[fuse_begin + f].part
  int32_t fuse_begin, fuse_count;
};

// One TR_MM op folded into the GEMM that produces its later operand (trace fusion).
struct DfFused {
  int32_t tmap;           // tensor map 2*tmap: the other operand [Lt][N][N], 8 x 32 boxes
  int32_t tiles;          // output tiles per time slice of the host GEMM
  double2* part;          // [Lt][tiles][8 warps] complex partials
  double2* root;          // root values [Lt] of the TR's tree (written by the finish kernel)
};

struct DfQueue {
  const DfOp* ops;
  const int32_t* item_op;    // op index of each item
  const int32_t* item_local; // index of each item within its op (queue order need not be op-major)
  int32_t n_ops;
  int64_t n_items;
  unsigned long long* head;  // atomic queue head (zeroed per launch)
};

struct DfArgs {
  const DfFused* fused;       // fused traces of GEMM ops
  DfQueue q;                  // GEMM items
  DfQueue qt;                 // TR_MM items
  const int32_t* dep_slot;    // sync slot an op waits on
  const int32_t* dep_target;  // value the slot must reach; -C: a copy in C time-slice chunks,
                              // the item needs the chunk holding its slice (value chunk+1);
                              // <= -2^20: per-slice GEMM counter, slot + slice must reach
                              // -target - 2^20 (the op's items per time slice)
  const void* tmaps;          // CUtensorMap array (64-byte aligned, global memory)
  int* sync;                  // done counters + copy flags (zeroed per launch)
  unsigned long long* prof;   // optional: per GEMM item {claim, ready, end, smid, first data, loop end, kind, -}
  unsigned long long* prof_t; // optional: the same per TR_MM item
  long long* prof_sm;         // optional: per CTA {wait cycles G/T, work cycles G/T, stages G/T, smid, -}
  int32_t ahead_g, ahead_t;   // items a CTA may hold claimed-but-unpublished per queue (<= 4)
  int32_t Lt;                 // time slices (chunked-copy targets)
};

cudaError_t df_preload();
// Launch the persistent worker (stream-ordered; the sync area must be zero).
cudaError_t df_launch(const DfArgs& a, int grid, cudaStream_t s);
// Tile / chunk geometry the builder needs (matches the worker's Cfg).
void df_gemm_tile_dims(int* BM, int* BN, int* BK, int* slot_doubles);
int df_trace_block();
// fused traces need GEMM stages that hold a half partner tile (32 KB)
bool df_supports_fusion();
// Encode the TMA maps of one GEMM problem into dst[0] (A) and dst[1] (B).
bool df_encode_maps(void* dst, const void* A, const void* B, int64_t M, int64_t Nn, int64_t Kin, int64_t Ko,
                    int64_t batch, int64_t lda, int64_t sAo, int64_t sAb, int64_t ldb, int64_t sBo, int64_t sBb);
// TMA maps of a TR_MM op's operands ([Lt][N][N] complex, 32-row boxes); *chunk_wide is set
// when the maps cover a whole 32x32 block per box (N % 8 == 0).
bool df_encode_trace_maps(void* dst, const void* A, const void* B, int64_t Lt, int64_t N, int32_t* chunk_wide);
// TMA maps of a BB3 op's operands (baryons [Lt][S][N][N][N] as 4-d tensors (k, j, i, t S + s):
// boxes of 8 complex x 1 x 32 rows, so a stage holds the same 32x32 sub-matrix block pair).
bool df_encode_bb3_maps(void* dst, const void* A, const void* B, int64_t Lt, int64_t N, int64_t S);
// TMA map of a fused trace's other operand ([Lt][N][N] complex, boxes of 8 complex x 32 rows).
bool df_encode_partner_map(void* dst, const void* X, int64_t Lt, int64_t N);
// root[t] = sum over tiles, warps of part[t][tile][warp] (fixed order), for every fused trace.
cudaError_t df_launch_fused_finish(const DfFused* fused, int32_t n_fused, int64_t Lt, cudaStream_t s);

}  // namespace cc
