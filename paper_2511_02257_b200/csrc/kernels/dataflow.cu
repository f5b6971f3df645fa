// Persistent dataflow worker for a whole plan (see dataflow.hpp for the protocol).
//
// One CTA per SM: 8 consumer warps + 1 producer warp.  The producer takes the plan's work
// items from one queue in plan order, decodes them, waits for their dependencies and streams
// their operands through a STAGES-deep TMA ring of 32 KB stages:
//   GEMM item (MM1/BM1/BB2 output tile, or one k-chunk of it): one stage per 16-complex
//     k-tile (A 64x16 + B 16x64 complex), consumed by the FP64 DMMA k-tile step
//     (common.cuh, 64 x 64 complex CTA tile, warp tile 32 x 16);
//   TR_MM item (a range of 32x32 block pairs of one time slice): one stage per block pair
//     (A[t,I,J] and B[t,J,I], 16 KB each, 128-byte swizzled), consumed with FP64 FMAs.
// Decoded items reach the consumers through a small ring of ItemInfo slots guarded by
// mbarriers, so queue latency, dependency checks and pipeline fill of item n+1 overlap the
// math of item n.  The same warps issue the DMMAs and the trace FMAs: both run on the SM's
// FP64 datapath, where a co-resident DFMA kernel is starved by DMMA issue (measured:
// tools/microbench/dmma_dfma_share.cu); the trace operands stream in by TMA behind the GEMM
// work instead.
// Reductions are deterministic: a chunked tile is summed chunk by chunk by the CTA that
// completes its last chunk (ticket); a trace slice's pieces are summed in piece order by the
// CTA that completes its last piece; CTA partials use fixed shuffle trees.  Completion is
// published with a consumer barrier, one release fence and one atomic increment of the op's
// done counter; the producer acquires it (ld.acquire.gpu) and issues a proxy fence before TMA
// reads data other SMs wrote with ordinary stores.
#include "common.cuh"
#include "dataflow.hpp"
#include "kernels.hpp"

namespace cc {
namespace {
using namespace dev;

using GC = Cfg<64, 64, 16, 32, 16, 5>;     // 5 x 32 KB stages
constexpr int CW = GC::NCW * 32;           // 256 consumer threads (+ producer warp + publisher warp)
constexpr int NT = CW + 64;
constexpr int TB = 32;                     // trace block edge (complex)
constexpr int INFO = 4;                    // decoded items in flight producer -> consumers
static_assert(GC::A_BYTES == TB * TB * 16 && GC::B_BYTES == TB * TB * 16, "a trace block pair fills one stage");

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

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ double2 cmul_acc(double2 acc, double2 x, double2 y) {
  acc.x = fma(x.x, y.x, acc.x);
  acc.x = fma(-x.y, y.y, acc.x);
  acc.y = fma(x.x, y.y, acc.y);
  acc.y = fma(x.y, y.x, acc.y);
  return acc;
}

// One work item as the producer decoded it (shared memory, handed to the consumers).
struct ItemInfo {
  int64_t item;           // >= n_items: stop
  int64_t tile;           // GEMM
  const void* tA;
  const void* tB;
  int32_t op, kind, npos; // npos: stages the item consumes
  int32_t tm, tn, b, k0, kt_per_o, chunk;   // GEMM
  int32_t t, u0, nb, piece;                 // TRACE
  unsigned long long t_disp, t_ready;       // profiling (producer)
  unsigned long long t_start, t_first, t_comp;  // profiling (consumers)
};

// Decode `item` (hint: the op of the previous item; consecutive items usually share it).
__device__ __forceinline__ int decode_item(const DfArgs& a, int64_t item, ItemInfo& inf, int hint) {
  inf.item = item;
  if (item >= a.q.n_items) return hint;
  int oi = hint;
  if (oi < 0 || item < a.q.ops[oi].first_item || item >= a.q.ops[oi].first_item + a.q.ops[oi].n_items)
    oi = find_op(a.q, item);
  const DfOp& op = a.q.ops[oi];
  const int64_t local = item - op.first_item;
  inf.op = oi;
  inf.kind = op.kind;
  inf.tA = static_cast<const uint8_t*>(a.tmaps) + size_t(2 * op.tmap) * 128;
  inf.tB = static_cast<const uint8_t*>(a.tmaps) + size_t(2 * op.tmap + 1) * 128;
  if (op.kind == 0) {
    const int64_t tile = local / op.n_chunks;
    const int chunk = int(local - tile * op.n_chunks);
    const int64_t tiles_mn = int64_t(op.tiles_m) * op.tiles_n;
    const int64_t b = tile / tiles_mn;
    const int64_t rr = tile - b * tiles_mn;
    inf.tile = tile;
    inf.chunk = chunk;
    inf.tn = int(rr / op.tiles_m);
    inf.tm = int(rr - int64_t(inf.tn) * op.tiles_m);
    inf.b = int(b);
    inf.k0 = int((int64_t(chunk) * op.KT) / op.n_chunks);
    inf.npos = int((int64_t(chunk + 1) * op.KT) / op.n_chunks) - inf.k0;
    inf.kt_per_o = op.kt_per_o;
  } else {
    const int t = int(local / op.P), p = int(local - int64_t(t) * op.P);
    const int U = op.nb * op.nb;
    inf.t = t;
    inf.piece = p;
    inf.nb = op.nb;
    inf.u0 = int((int64_t(p) * U) / op.P);
    inf.npos = int((int64_t(p + 1) * U) / op.P) - inf.u0;
  }
  return oi;
}

// launch bounds of 12 warps although 10 run: caps registers at 168 (3 warps per SM
// sub-partition x 32 x 168 <= 16K registers each)
__global__ void __launch_bounds__(CW + 128, 1) df_worker(DfArgs a) {
  using C = GC;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned stage base, derived from the __shared__ array by pointer arithmetic so
  // the compiler keeps the shared address space (LDS, not generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  __shared__ ItemInfo s_info[INFO];
  __shared__ uint64_t info_full[INFO], info_empty[INFO];
  __shared__ double2 red[GC::NCW];
  __shared__ int s_flag;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    for (int s = 0; s < INFO; ++s) {
      mbar_init(&info_full[s], 1);
      mbar_init(&info_empty[s], 1);    // released by the publisher warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == C::NCW) {
    // --------------------------------- producer -------------------------------------------
    if (lane != 0) return;
    uint32_t pos = 0;   // ring positions issued
    int hint = -1;
    for (uint32_t n = 0;; ++n) {
      const int slot = int(n % INFO);
      mbar_wait(&info_empty[slot], ((n / INFO) & 1u) ^ 1u);
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
      mbar_arrive(&info_full[slot]);   // release: the decoded item is visible to the consumers
      if (stop) break;
      for (int k = 0; k < inf.npos; ++k, ++pos) {
        const int st = int(pos % C::STAGES);
        mbar_wait(&empty[st], ((pos / C::STAGES) & 1u) ^ 1u);
        mbar_expect_tx(&full[st], C::STAGE_BYTES);
        uint8_t* sA = smem + st * C::STAGE_BYTES;
        uint8_t* sB = sA + C::A_BYTES;
        if (inf.kind == 0) {
          const int kk = inf.k0 + k;
          const int ko = kk / inf.kt_per_o;
          const int ki0 = (kk - ko * inf.kt_per_o) * C::BK;
#pragma unroll
          for (int kc = 0; kc < C::BK / 8; ++kc)
            tma_load_4d_g(sA + kc * C::BM * 128, inf.tA, &full[st], 2 * (ki0 + kc * 8), inf.tm * C::BM, ko, inf.b);
#pragma unroll
          for (int nc = 0; nc < C::BN / 8; ++nc)
            tma_load_4d_g(sB + nc * C::BK * 128, inf.tB, &full[st], 2 * (inf.tn * C::BN + nc * 8), ki0, ko, inf.b);
        } else {
          const int u = inf.u0 + k;
          const int I = u / inf.nb, J = u - I * inf.nb;
#pragma unroll
          for (int ch = 0; ch < TB / 8; ++ch) {  // A[t, I*32 + r, J*32 + 8ch + s] and B[t, J*32 + r, I*32 + 8ch + s]
            tma_load_4d_g(sA + ch * TB * 128, inf.tA, &full[st], 2 * (J * TB + 8 * ch), I * TB, 0, inf.t);
            tma_load_4d_g(sB + ch * TB * 128, inf.tB, &full[st], 2 * (I * TB + 8 * ch), J * TB, 0, inf.t);
          }
        }
      }
    }
    return;
  }
  if (warp == C::NCW + 1) {
    // --------------------------------- publisher ------------------------------------------
    // Completion of item n: the consumers arrive on named barrier 2 + slot after their last
    // store and go on with item n+1; this warp syncs on it (acquiring their stores), makes
    // them visible at GPU scope (cumulative fence) and bumps the op's done counter — the
    // fence's drain latency leaves the consumers' critical path.  A slot (and its barrier)
    // is reused only after this warp releases info_empty, so at most INFO items are pending.
    for (uint32_t n = 0;; ++n) {
      const int slot = int(n % INFO);
      mbar_wait(&info_full[slot], (n / INFO) & 1u);
      const ItemInfo& cur = s_info[slot];
      const int64_t item = cur.item;
      if (item >= a.q.n_items) break;
      asm volatile("bar.sync %0, %1;" ::"r"(2 + slot), "r"(CW + 32) : "memory");
      if (lane == 0) {
        __threadfence();
        atomicAdd(a.sync + a.q.ops[cur.op].sync_id, 1);
        if (a.prof) {
          unsigned long long* pr = a.prof + 8 * item;
          pr[0] = cur.t_disp;
          pr[1] = cur.t_ready;
          pr[2] = gtimer();
          pr[3] = smid();
          pr[4] = cur.t_start;
          pr[5] = cur.t_comp;
          pr[6] = cur.kind;
          pr[7] = cur.t_first;
        }
        mbar_arrive(&info_empty[slot]);
      }
      __syncwarp();
    }
    return;
  }

  // ----------------------------------- consumers ---------------------------------------------
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int g = lane >> 2, t = lane & 3;
  const bool q = (g & 1) != 0;
  uint32_t ring = 0;
  for (uint32_t n = 0;; ++n) {
    const int slot = int(n % INFO);
    mbar_wait(&info_full[slot], (n / INFO) & 1u);
    const ItemInfo& cur = s_info[slot];
    const int64_t item = cur.item;
    if (item >= a.q.n_items) break;
    const DfOp& op = a.q.ops[cur.op];
    const int npos = cur.npos;
    unsigned long long t_first = 0, t_comp = 0;
    const unsigned long long t_start = (tid == 0 && a.prof) ? gtimer() : 0ull;

    if (cur.kind == 0) {
      // ---------------- GEMM tile (or k-chunk of a tile) ----------------
      double acc[C::MI][C::NI][2];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int k = 0; k < C::NI; ++k) acc[i][k][0] = acc[i][k][1] = 0.0;
      for (int i = 0; i < npos; ++i) {
        const uint32_t r = ring + i;
        const int st = int(r % C::STAGES);
        mbar_wait(&full[st], (r / C::STAGES) & 1u);
        if (i == 0 && tid == 0 && a.prof) t_first = gtimer();
        const uint8_t* sA = smem + st * C::STAGE_BYTES;
        dmma_ktile<C>(sA, sA + C::A_BYTES, wm, wn, g, t, q, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      ring += npos;
      if (tid == 0 && a.prof) t_comp = gtimer();
      const int64_t tile = cur.tile;
      const int chunk = cur.chunk;
      double2* out = static_cast<double2*>(op.C) + int64_t(cur.b) * op.sCb;
      bool store = true;
      if (op.n_chunks > 1) {
        // publish this chunk's partial; the CTA completing the tile's last chunk sums them
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
        named_sync(1, CW);
        if (tid == 0) {
          const int old = atomicAdd(&op.tile_cnt[tile], 1);
          s_flag = (old == op.n_chunks - 1);
          if (s_flag) op.tile_cnt[tile] = 0;
        }
        named_sync(1, CW);
        store = s_flag != 0;
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
          const int64_t row = int64_t(cur.tm) * C::BM + wm * C::WM + i * 8 + g;
          if (row >= op.M) continue;
#pragma unroll
          for (int k = 0; k < C::NI; ++k) {
            const int64_t col = int64_t(cur.tn) * C::BN + wn * C::WN + k * 4 + t;
            if (col < op.Nn) out[row * op.ldc + col] = make_double2(acc[i][k][0], acc[i][k][1]);
          }
        }
      }
    } else {
      // ---------------- TR_MM piece: sum over block pairs of A[r][c] * B[c][r] ----------------
      double2 acc = make_double2(0.0, 0.0);
      for (int i = 0; i < npos; ++i) {
        const uint32_t r = ring + i;
        const int st = int(r % C::STAGES);
        mbar_wait(&full[st], (r / C::STAGES) & 1u);
        if (i == 0 && tid == 0 && a.prof) t_first = gtimer();
        const uint8_t* sA = smem + st * C::STAGE_BYTES;
        const uint8_t* sB = sA + C::A_BYTES;
        // element (row, col) of a 32x32 block: chunk col/8, 128-byte row `row`, 16-byte slot
        // (col%8) ^ (row%8) (TMA 128-byte swizzle); warp w takes rows w, w+8, w+16, w+24 of A,
        // lane = column c: A[r][c] row-contiguous, B[c][r] one 128-byte row per lane — both
        // conflict-free.
#pragma unroll
        for (int qq = 0; qq < TB / 8; ++qq) {
          const int rr = warp + qq * 8, c = lane;
          const double2 av = *reinterpret_cast<const double2*>(sA + (c >> 3) * (TB * 128) + rr * 128 +
                                                               (((c & 7) ^ (rr & 7)) << 4));
          const double2 bv = *reinterpret_cast<const double2*>(sB + (rr >> 3) * (TB * 128) + c * 128 +
                                                               (((rr & 7) ^ (c & 7)) << 4));
          acc = cmul_acc(acc, av, bv);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      ring += npos;
      if (tid == 0 && a.prof) t_comp = gtimer();
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) red[warp] = acc;
      named_sync(1, CW);
      double2* outp = static_cast<double2*>(op.out);
      if (tid == 0) {
        double2 s = red[0];
        for (int w = 1; w < C::NCW; ++w) {
          s.x += red[w].x;
          s.y += red[w].y;
        }
        if (op.P == 1) {
          outp[cur.t] = s;
          s_flag = 0;
        } else {
          static_cast<double2*>(op.tr_part)[int64_t(cur.t) * op.P + cur.piece] = s;
          __threadfence();
          const int ticket = atomicAdd(&op.tr_cnt[cur.t], 1);
          s_flag = (ticket == op.P - 1);
          if (s_flag) op.tr_cnt[cur.t] = 0;
        }
      }
      named_sync(1, CW);
      if (s_flag && warp == 0) {
        // the last piece of slice t: fixed-order sum of the P pieces
        __threadfence();
        const double* pp = static_cast<const double*>(op.tr_part) + 2 * int64_t(cur.t) * op.P;
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
        if (lane == 0) outp[cur.t] = make_double2(sx, sy);
      }
    }

    if (tid == 0 && a.prof) {
      ItemInfo& w = s_info[slot];
      w.t_start = t_start;
      w.t_first = t_first;
      w.t_comp = t_comp;
    }
    // release the item to the publisher (barrier arrive orders this thread's stores before it)
    asm volatile("bar.arrive %0, %1;" ::"r"(2 + slot), "r"(CW + 32) : "memory");
  }
}

}  // namespace

cudaError_t df_preload() {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, df_worker);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(df_worker, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::SMEM);
  return e;
}

void df_gemm_tile_dims(int* BM, int* BN, int* BK, int* slot_doubles) {
  *BM = GC::BM;
  *BN = GC::BN;
  *BK = GC::BK;
  *slot_doubles = GC::SLOT_DOUBLES;
}

int df_trace_block() { return TB; }

cudaError_t df_launch(const DfArgs& a, int grid, cudaStream_t s) {
  df_worker<<<grid, NT, GC::SMEM, s>>>(a);
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

bool df_encode_trace_maps(void* dst, const void* A, const void* B, int64_t Lt, int64_t N) {
  // A, B as [Lt][N rows][N complex]: boxes of 32 rows x 8 complex (128-byte swizzle)
  ZgemmProblem p{};
  p.A = A;
  p.B = B;
  p.M = N;
  p.Nn = N;
  p.Kin = N;
  p.Ko = 1;
  p.batch = Lt;
  p.lda = N;
  p.sAb = N * N;
  p.ldb = N;
  p.sBb = N * N;
  return encode_zgemm_maps(dst, static_cast<uint8_t*>(dst) + 128, p, TB, TB);
}

}  // namespace cc
