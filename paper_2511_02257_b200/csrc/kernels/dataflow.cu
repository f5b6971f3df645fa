// Persistent dataflow workers for a whole plan (see dataflow.hpp for the protocol).
//
// gemm_worker: one CTA per SM, 8 DMMA warps (warp tile 32 rows x 16 complex, CTA tile
//   64 x 64 complex); thread 0 also drives the TMA ring (prefetch distance STAGES-1 k-tiles,
//   refilled as soon as every warp released the previous stage).  An item is one output
//   tile, or one k-chunk of a tile for ops with few tiles (BB2); the CTA that completes the
//   last chunk of a tile (ticket) sums the chunk partials in chunk order — deterministic.
//   Register cap 192 so a trace-worker CTA fits on the same SM.
// trace_worker: 256 threads, <= 64 registers, 66 KB of shared memory: streams its (t, piece)
//   unit range through a 2-stage cp.async ring (L2-only copies: operands were written by other
//   SMs during this launch), fixed-order reductions, last-piece finisher per time slice.
// Both publish completion with per-thread fences, a CTA barrier and one atomic increment
// of the op's done counter; waiters spin with ld.acquire.gpu and issue a proxy fence
// before TMA reads data other SMs wrote with ordinary stores.
#include "common.cuh"
#include "dataflow.hpp"
#include "kernels.hpp"

namespace cc {
namespace {
using namespace dev;

using GC = Cfg<64, 64, 16, 32, 16, 3>;   // same tile math as zgemm; 3 stages leave shared memory
                                         // for a 4-stage trace worker on the SM
constexpr int GW_THREADS = GC::NCW * 32;  // 256 consumer threads (+1 producer warp)
constexpr int TR_TB = 32;
constexpr int TR_THREADS = 128;   // 4 warps: one per SM sub-partition (see gemm_worker)
constexpr int TR_WARPS = TR_THREADS / 32;

__device__ __forceinline__ void tma_load_4d_g(void* dst, const void* map, uint64_t* bar, int c0, int c1, int c2,
                                              int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ int find_op(const DfQueue& q, int64_t item) {
  int lo = 0, hi = q.n_ops - 1;
  while (lo < hi) {  // last op with first_item <= item
    const int mid = (lo + hi + 1) >> 1;
    if (q.ops[mid].first_item <= item) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void wait_deps(const DfArgs& a, const DfOp& op) {
  for (int d = 0; d < op.dep_count; ++d) {
    const int* slot = a.sync + a.dep_slot[op.dep_begin + d];
    const int target = a.dep_target[op.dep_begin + d];
    while (ld_acquire(slot) < target) __nanosleep(64);
  }
}

// ---------------------------------------------------------------------------------------------
// One GEMM item as the producer decoded it (shared memory, handed to the consumer warps).
struct ItemInfo {
  int64_t item;          // >= n_items: stop
  int64_t tile;
  const void* tA;
  const void* tB;
  int32_t op, tm, tn, b, k0, nk, kt_per_o, chunk;
  unsigned long long t_disp, t_ready;   // profiling
};

// Decode `item` (hint: the op of the previous item — consecutive items usually share it,
// which skips the binary search over the op table).
__device__ __forceinline__ int decode_item(const DfArgs& a, int64_t item, ItemInfo& inf, int hint) {
  inf.item = item;
  if (item >= a.q.n_items) return hint;
  int oi = hint;
  if (oi < 0 || item < a.q.ops[oi].first_item || item >= a.q.ops[oi].first_item + a.q.ops[oi].n_items)
    oi = find_op(a.q, item);
  const DfOp& op = a.q.ops[oi];
  const int64_t local = item - op.first_item;
  const int64_t tile = local / op.n_chunks;
  const int chunk = int(local - tile * op.n_chunks);
  const int64_t tiles_mn = int64_t(op.tiles_m) * op.tiles_n;
  const int64_t b = tile / tiles_mn;
  const int64_t rr = tile - b * tiles_mn;
  inf.op = oi;
  inf.tile = tile;
  inf.chunk = chunk;
  inf.tn = int(rr / op.tiles_m);
  inf.tm = int(rr - int64_t(inf.tn) * op.tiles_m);
  inf.b = int(b);
  inf.k0 = int((int64_t(chunk) * op.KT) / op.n_chunks);
  inf.nk = int((int64_t(chunk + 1) * op.KT) / op.n_chunks) - inf.k0;
  inf.kt_per_o = op.kt_per_o;
  inf.tA = static_cast<const uint8_t*>(a.tmaps) + size_t(2 * op.tmap) * 128;
  inf.tB = static_cast<const uint8_t*>(a.tmaps) + size_t(2 * op.tmap + 1) * 128;
  return oi;
}

constexpr int GW_INFO = 4;   // decoded items in flight between producer and consumers

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Persistent DMMA worker: 8 consumer warps (DMMA) + 1 producer warp.  The producer takes
// items from the queue, decodes them, waits for their dependencies and streams their TMA
// k-tiles through the STAGES ring; decoded items reach the consumers through a small ring of
// ItemInfo slots guarded by mbarriers.  Queue latency, dependency checks and pipeline fill of
// item n+1 thus overlap the DMMA work and epilogue of item n.  Only the producer ever waits
// on dependencies, and only for items no consumer has started, so the no-deadlock argument of
// dataflow.hpp holds.
// Register budget: the SM's register file is split over 4 sub-partitions (warp w on w % 4),
// 16K registers each; with 9 warps here sub-partition 0 holds 3 of them, so 152 registers per
// thread leave exactly one 56-register warp of the 4-warp trace worker room on every
// sub-partition (3*32*152 + 32*56 = 16384): the two workers co-reside on each SM.
__global__ void __maxnreg__(152) gemm_worker(DfArgs a) {
  using C = GC;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned stage base, derived from the __shared__ array by pointer arithmetic so
  // the compiler keeps the shared address space (LDS, not generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  __shared__ ItemInfo s_info[GW_INFO];
  __shared__ uint64_t info_full[GW_INFO], info_empty[GW_INFO];
  __shared__ int s_fin;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    for (int s = 0; s < GW_INFO; ++s) {
      mbar_init(&info_full[s], 1);
      mbar_init(&info_empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == C::NCW) {
    // ------------------------------- producer -------------------------------------------
    if (lane != 0) return;
    uint32_t pos = 0;   // ring positions issued
    int hint = -1;
    for (uint32_t n = 0;; ++n) {
      const int slot = int(n % GW_INFO);
      mbar_wait(&info_empty[slot], ((n / GW_INFO) & 1u) ^ 1u);
      ItemInfo& inf = s_info[slot];
      const unsigned long long t0 = a.prof ? gtimer() : 0ull;
      hint = decode_item(a, int64_t(atomicAdd(a.q.head, 1ull)), inf, hint);
      const bool stop = inf.item >= a.q.n_items;
      if (!stop) {
        wait_deps(a, a.q.ops[inf.op]);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(inf.tA) : "memory");
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(inf.tB) : "memory");
      }
      inf.t_disp = t0;
      inf.t_ready = a.prof ? gtimer() : 0ull;
      mbar_arrive(&info_full[slot]);   // release: the info is visible to the consumers
      if (stop) break;
      for (int k = 0; k < inf.nk; ++k, ++pos) {
        const int st = int(pos % C::STAGES);
        mbar_wait(&empty[st], ((pos / C::STAGES) & 1u) ^ 1u);
        mbar_expect_tx(&full[st], C::STAGE_BYTES);
        uint8_t* sA = smem + st * C::STAGE_BYTES;
        uint8_t* sB = sA + C::A_BYTES;
        const int kk = inf.k0 + k;
        const int ko = kk / inf.kt_per_o;
        const int ki0 = (kk - ko * inf.kt_per_o) * C::BK;
#pragma unroll
        for (int kc = 0; kc < C::BK / 8; ++kc)
          tma_load_4d_g(sA + kc * C::BM * 128, inf.tA, &full[st], 2 * (ki0 + kc * 8), inf.tm * C::BM, ko, inf.b);
#pragma unroll
        for (int nc = 0; nc < C::BN / 8; ++nc)
          tma_load_4d_g(sB + nc * C::BK * 128, inf.tB, &full[st], 2 * (inf.tn * C::BN + nc * 8), ki0, ko, inf.b);
      }
    }
    return;
  }

  // --------------------------------- consumers ---------------------------------------------
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int g = lane >> 2, t = lane & 3;
  const bool q = (g & 1) != 0;
  uint32_t ring = 0;
  for (uint32_t n = 0;; ++n) {
    const int slot = int(n % GW_INFO);
    mbar_wait(&info_full[slot], (n / GW_INFO) & 1u);
    const ItemInfo& cur = s_info[slot];
    const int64_t item = cur.item;
    if (item >= a.q.n_items) break;
    const DfOp& op = a.q.ops[cur.op];
    const int nk = cur.nk;
    unsigned long long t_first = 0, t_comp = 0;

    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int k = 0; k < C::NI; ++k) acc[i][k][0] = acc[i][k][1] = 0.0;
    for (int i = 0; i < nk; ++i) {
      const uint32_t r = ring + i;
      const int st = int(r % C::STAGES);
      mbar_wait(&full[st], (r / C::STAGES) & 1u);
      if (i == 0 && tid == 0 && a.prof) t_first = gtimer();
      const uint8_t* sA = smem + st * C::STAGE_BYTES;
      dmma_ktile<C>(sA, sA + C::A_BYTES, wm, wn, g, t, q, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    ring += nk;
    if (tid == 0 && a.prof) t_comp = gtimer();

    const int64_t tile = cur.tile;
    const int chunk = cur.chunk;
    const int tm = cur.tm, tn = cur.tn;
    double2* out = static_cast<double2*>(op.C) + int64_t(cur.b) * op.sCb;
    bool store = true;
    if (op.n_chunks > 1) {
      // publish this chunk's partial, then the last chunk of the tile sums all of them
      double* base = static_cast<double*>(op.part) + (tile * op.n_chunks) * int64_t(C::SLOT_DOUBLES);
      double* mine = base + int64_t(chunk) * C::SLOT_DOUBLES + warp * (C::FRAG * 32);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int k = 0; k < C::NI; ++k) {
          __stcg(mine + ((i * C::NI + k) * 2 + 0) * 32 + lane, acc[i][k][0]);
          __stcg(mine + ((i * C::NI + k) * 2 + 1) * 32 + lane, acc[i][k][1]);
        }
      __threadfence();
      named_sync(1, GW_THREADS);
      if (tid == 0) {
        const int old = atomicAdd(&op.tile_cnt[tile], 1);
        s_fin = (old == op.n_chunks - 1);
        if (s_fin) op.tile_cnt[tile] = 0;
      }
      named_sync(1, GW_THREADS);
      store = s_fin != 0;
      if (store) {
        __threadfence();
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int k = 0; k < C::NI; ++k) acc[i][k][0] = acc[i][k][1] = 0.0;
        for (int c = 0; c < op.n_chunks; ++c) {
          const double* src = base + int64_t(c) * C::SLOT_DOUBLES + warp * (C::FRAG * 32);
#pragma unroll
          for (int i = 0; i < C::MI; ++i)
#pragma unroll
            for (int k = 0; k < C::NI; ++k) {
              acc[i][k][0] += __ldcg(src + ((i * C::NI + k) * 2 + 0) * 32 + lane);
              acc[i][k][1] += __ldcg(src + ((i * C::NI + k) * 2 + 1) * 32 + lane);
            }
        }
      }
    }
    if (store) {
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const int64_t row = int64_t(tm) * C::BM + wm * C::WM + i * 8 + g;
        if (row >= op.M) continue;
#pragma unroll
        for (int k = 0; k < C::NI; ++k) {
          const int64_t col = int64_t(tn) * C::BN + wn * C::WN + k * 4 + t;
          if (col < op.Nn) out[row * op.ldc + col] = make_double2(acc[i][k][0], acc[i][k][1]);
        }
      }
    }
    named_sync(1, GW_THREADS);
    if (tid == 0) {
      __threadfence();   // cumulative: the consumers' stores (ordered by the barrier) before the count
      atomicAdd(a.sync + op.sync_id, 1);
      if (a.prof) {
        unsigned long long* pr = a.prof + 8 * item;
        pr[0] = cur.t_disp;
        pr[1] = cur.t_ready;
        pr[2] = gtimer();
        pr[3] = smid();
        pr[4] = t_first;
        pr[5] = t_comp;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&info_empty[slot]);
  }
}

// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double2 cmul_acc(double2 acc, double2 x, double2 y) {
  acc.x = fma(x.x, y.x, acc.x);
  acc.x = fma(-x.y, y.y, acc.x);
  acc.y = fma(x.x, y.y, acc.y);
  acc.y = fma(x.y, y.x, acc.y);
  return acc;
}

// trace unit = 32x32 complex block A[t, I, J] and its partner B[t, J, I], staged in shared
// memory by cp.async (16-byte L2-only copies, zero-filled outside N), TR_STAGES deep, so the
// next units stream in without holding registers.  B is read transposed (lane = row), so its
// 16-byte element (r, c) is stored at column c ^ (r & 7): the 8 lanes of a shared-memory
// phase then hit 8 different 16-byte bank groups (conflict-free, no padding).
constexpr int TR_STAGES = 3;
constexpr int TR_A_BYTES = TR_TB * TR_TB * 16;
constexpr int TR_B_BYTES = TR_TB * TR_TB * 16;   // XOR-swizzled (see below)
constexpr int TR_SMEM = TR_STAGES * (TR_A_BYTES + TR_B_BYTES);

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned d = smem_u32(dst);
  const int n = valid ? 16 : 0;   // src-size 0: the 16 bytes are zero-filled
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Issue the copies of unit u of slice (At, Bt) into stage st (every thread: 4 + 4 chunks).
__device__ __forceinline__ void tr_issue(uint8_t* smem, int st, const double2* At, const double2* Bt, int64_t N,
                                         int nb, int u, int tid) {
  const int I = u / nb, J = u - I * nb;
  const int64_t i0 = int64_t(I) * TR_TB, j0 = int64_t(J) * TR_TB;
  double2* sA = reinterpret_cast<double2*>(smem + st * (TR_A_BYTES + TR_B_BYTES));
  double2* sB = reinterpret_cast<double2*>(smem + st * (TR_A_BYTES + TR_B_BYTES) + TR_A_BYTES);
#pragma unroll
  for (int q = 0; q < 1024 / TR_THREADS; ++q) {
    const int e = tid + q * TR_THREADS;   // 0..1023: row e/32, column e%32
    const int r = e >> 5, c = e & 31;
    const int64_t ia = i0 + r, ja = j0 + c;   // A[t, I0 + r, J0 + c]
    const int64_t jb = j0 + r, ib = i0 + c;   // B[t, J0 + r, I0 + c]
    const bool va = ia < N && ja < N, vb = jb < N && ib < N;
    cp_async16(sA + r * TR_TB + c, va ? At + ia * N + ja : At, va);
    cp_async16(sB + r * TR_TB + (c ^ (r & 7)), vb ? Bt + jb * N + ib : Bt, vb);
  }
}

__global__ void __maxnreg__(56) trace_worker(DfArgs a) {
  extern __shared__ __align__(16) uint8_t tr_smem[];
  __shared__ double2 red[TR_THREADS / 32];
  __shared__ int64_t s_item;
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.q.head, 1ull);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= a.q.n_items) break;
    const DfOp& op = a.q.ops[find_op(a.q, item)];
    unsigned long long t_disp = 0, t_ready = 0;
    if (tid == 0) {
      if (a.prof) t_disp = gtimer();
      wait_deps(a, op);
      if (a.prof) t_ready = gtimer();
    }
    __syncthreads();
    const int64_t local = item - op.first_item;
    const int t = int(local / op.P), p = int(local - int64_t(t) * op.P);
    const int U = op.nb * op.nb;
    const int u0 = int((int64_t(p) * U) / op.P), u1 = int((int64_t(p + 1) * U) / op.P);
    const int64_t N = op.N;
    const double2* At = static_cast<const double2*>(op.A) + int64_t(t) * N * N;
    const double2* Bt = static_cast<const double2*>(op.B) + int64_t(t) * N * N;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int s = 0; s < TR_STAGES; ++s) {
      if (u0 + s < u1) tr_issue(tr_smem, s, At, Bt, N, op.nb, u0 + s, tid);
      cp_async_commit();
    }
    for (int u = u0; u < u1; ++u) {
      const int st = (u - u0) % TR_STAGES;
      cp_async_wait<TR_STAGES - 1>();
      __syncthreads();
      const double2* sA = reinterpret_cast<const double2*>(tr_smem + st * (TR_A_BYTES + TR_B_BYTES));
      const double2* sB = reinterpret_cast<const double2*>(tr_smem + st * (TR_A_BYTES + TR_B_BYTES) + TR_A_BYTES);
#pragma unroll
      for (int q = 0; q < TR_TB / TR_WARPS; ++q) {
        const int r = warp + q * TR_WARPS;
        acc = cmul_acc(acc, sA[r * TR_TB + lane], sB[lane * TR_TB + (r ^ (lane & 7))]);  // A[I0+r][J0+lane] B[J0+lane][I0+r]
      }
      __syncthreads();
      if (u + TR_STAGES < u1) tr_issue(tr_smem, st, At, Bt, N, op.nb, u + TR_STAGES, tid);
      cp_async_commit();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    double2* outp = static_cast<double2*>(op.out);
    if (tid == 0) {
      double2 s = red[0];
      for (int w = 1; w < TR_THREADS / 32; ++w) {
        s.x += red[w].x;
        s.y += red[w].y;
      }
      if (op.P == 1) {
        outp[t] = s;
        s_last = 0;
      } else {
        static_cast<double2*>(op.tr_part)[int64_t(t) * op.P + p] = s;
        __threadfence();
        const int ticket = atomicAdd(&op.tr_cnt[t], 1);
        s_last = (ticket == op.P - 1);
      }
    }
    __syncthreads();
    if (s_last && warp == 0) {
      __threadfence();
      const double* pp = static_cast<const double*>(op.tr_part) + 2 * int64_t(t) * op.P;
      double sx = 0.0, sy = 0.0;
      for (int k = lane; k < op.P; k += 32) {
        sx += __ldcg(pp + 2 * k);
        sy += __ldcg(pp + 2 * k + 1);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if (lane == 0) {
        outp[t] = make_double2(sx, sy);
        op.tr_cnt[t] = 0;
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      atomicAdd(a.sync + op.sync_id, 1);
      if (a.prof) {
        unsigned long long* pr = a.prof + 8 * item;
        pr[0] = t_disp;
        pr[1] = t_ready;
        pr[2] = gtimer();
        pr[3] = smid();
      }
    }
  }
}

}  // namespace

size_t df_gemm_smem_bytes() { return size_t(GC::SMEM); }

cudaError_t df_preload() {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, gemm_worker);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, trace_worker);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(gemm_worker, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::SMEM);
  // both workers ask for the largest shared-memory carveout, so an SM configured for a GEMM
  // worker (132 KB) still has room for a trace worker (17 KB): the two co-reside
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_worker, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(trace_worker, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(trace_worker, cudaFuncAttributeMaxDynamicSharedMemorySize, TR_SMEM);
  return e;
}

void df_gemm_tile_dims(int* BM, int* BN, int* BK, int* slot_doubles) {
  *BM = GC::BM;
  *BN = GC::BN;
  *BK = GC::BK;
  *slot_doubles = GC::SLOT_DOUBLES;
}

int df_trace_block() { return TR_TB; }

cudaError_t df_launch_gemm(const DfArgs& a, int grid, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_worker, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gemm_worker<<<grid, GW_THREADS + 32, GC::SMEM, s>>>(a);
  return cudaGetLastError();
}

cudaError_t df_launch_trace(const DfArgs& a, int grid, cudaStream_t s) {
  trace_worker<<<grid, TR_THREADS, TR_SMEM, s>>>(a);
  return cudaGetLastError();
}

bool df_encode_maps(void* dst, const void* A, const void* B, int64_t M, int64_t Nn, int64_t Kin, int64_t Ko,
                    int64_t batch, int64_t lda, int64_t sAo, int64_t sAb, int64_t ldb, int64_t sBo, int64_t sBb) {
  ZgemmProblem p{};
  p.A = A;
  p.B = B;
  p.M = M;
  p.Nn = Nn;
  p.Kin = Kin;
  p.Ko = Ko;
  p.batch = batch;
  p.lda = lda;
  p.sAo = sAo;
  p.sAb = sAb;
  p.ldb = ldb;
  p.sBo = sBo;
  p.sBb = sBb;
  return encode_zgemm_maps(dst, static_cast<uint8_t*>(dst) + 128, p, GC::BM, GC::BK);
}

}  // namespace cc
