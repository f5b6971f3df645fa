// MM1 / BM1 / BB2 on the 5th-generation tensor cores: complex-double C = A B per time slice by Ozaki
// splitting into INT8 slices, tcgen05.mma kind::i8 with INT32 accumulators in TMEM, and an
// FP64 epilogue (reading V-6 in DESIGN.md).
//
// Why: sm_100a has no tcgen05 f64 kind (probed), so FP64 DMMA caps MM1 at 37 TF/s.  An INT8
// tcgen05 MMA is exact (integer products, INT32 accumulation), so a product of s-slice
// splittings reproduces the FP64 product to ~2^-7s relative to the row/column scale.
//
// Splitting (per time slice t):
//   A_cat = [Ar | Ai]              (N x 2N, row i scaled by 2^-eA[i], eA = max-exponent of row i)
//   B_cat = [[Br, Bi], [-Bi, Br]]  (2N x 2N, column c scaled by 2^-fB[c])
//   so that A_cat B_cat = [Cr | Ci]  (the real embedding of the complex product, 4M form)
//   x * 2^-e = sum_{k=0}^{s-1} 2^{-6-8k} x_k + r   (balanced base-256 digits of the fixed-point
//   value round(x 2^{6+8(s-1)})): x_0 in [-65, 65], x_k in [-128, 127], |r| <= 2^{-7-8(s-1)}.
//   C ~= 2^{eA+fB} sum_{i+j <= s-1} 2^{-12-8(i+j)} (A_i B_j)    (pairs below the anti-diagonal
//   cut are dropped, the standard Ozaki truncation); each pair is one signed kind::i8 MMA.
// Every (i, j) with i + j = d accumulates into one INT32 TMEM accumulator d (|acc| <= s 2^14 K
// < 2^31 for K = 2N <= 16384, s <= 7), so the epilogue sees s accumulators per output, converts
// each exactly to FP64 and sums them, most significant first.
//
// Layouts (device workspace, caller-owned):
//   SA int8: K-major rows of A_cat (Mp = roundup(M,128) rows, Kp = 2 Kc bytes, Kc =
//            roundup(K,32); K index: Re part at k, Im part at Kc + k), stored tile-contiguous
//            and pre-swizzled as [t][row block of 128][64-byte k chunk][slice][128][64]
//   SB int8: K-major rows of B_cat^T (2 Nc rows, Nc = roundup(Nn, BN/2); rows grouped per BN/2
//            output columns: row BN g + w, w < BN/2 -> Cr column (BN/2) g + w, else Ci), same
//            tiling with BN-row blocks
//   eA int32 [Lt][Mp], fB int32 [Lt][Nc]
// GEMM CTA (persistent): tiles of 128 rows x BN B_cat^T rows (BN = 64, or 96 for outputs >= 512
// columns: BN/2 complex output columns); a stage = all s slices of A and B for one 64-byte k
// chunk = contiguous bulk copies; one lane issues the tcgen05.mma's, 4 or 8 warps drain TMEM.
// BM1 / BB2 use the same kernels on their (two-level K) operand layouts; K is cut into chunks
// of 8192 complex terms (INT32 bound) whose FP64 partials are summed in order.  (A CTA-pair
// variant, cta_group::2 with M = 256 per instruction, measured slower in round 1: removed.)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <mutex>

#include "common.cuh"
#include "kernels.hpp"

namespace cc {
namespace oz {

constexpr int BM = 128;     // CTA rows (UMMA M)
constexpr int BKB = 64;     // K bytes per stage = one SWIZZLE_64B smem row (SW32 measured slower)
constexpr int UK = 32;      // K per kind::i8 MMA
constexpr int A_TILE = BM * BKB;    // 8 KB

// Tile width: BN B_cat^T rows per tile (UMMA N) = BN/2 complex output columns (Cr | Ci).
// 64 for small problems, 96 for wide ones (pick_bn): 1.5x the MACs per MMA instruction, the
// S diagonal accumulators then fill S*96 of the 512 TMEM columns (S <= 5).
template <int BN_>
struct Tile {
  static constexpr int BN = BN_;
  static constexpr int CG = BN_ / 2;                   // complex output columns per tile
  static constexpr int NEPI = BN_ > 64 ? 8 : 4;        // epilogue warps: lane quarters x column halves
  static constexpr int CPW = CG / (NEPI / 4);          // complex columns per epilogue warp
  static constexpr int B_TILE = BN_ * BKB;             // 4 / 6 KB
  // instruction descriptor kind::i8: D = S32 (bits 4-5 = 2), A, B signed (bits 7-9, 10-12 =
  // 1), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
  static constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN_ >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static_assert(BN_ == 64 || BN_ == 96, "tile width");
};
constexpr int SMEM_BUDGET = 222 * 1024;

template <int S, int BN>
struct Cfg {
  static constexpr int STAGE = S * (A_TILE + Tile<BN>::B_TILE);
  static constexpr int STAGES = (SMEM_BUDGET / STAGE) > 4 ? 4 : (SMEM_BUDGET / STAGE);
  static constexpr int SMEM = STAGES * STAGE + 1024;
  static_assert(STAGES >= 2, "too many slices for the stage budget");
  static_assert(S * BN <= 512, "accumulators exceed TMEM");
  static_assert(BN == 64 || BN == 96, "tile width");
};

struct Params {
  int Lt, Mp, Nc, Kp, Brows;      // Brows = rows of SB per (slice, t) = 2 Nc
  int M, Nn;                      // real output rows / complex columns
  int nch, kchs;                  // K chunks (split K for the INT32 bound) x stages per chunk
  long long ldc, sCb;             // C(t, m, n) at C + t sCb + m ldc + n (complex elements)
  const int* eA;
  const int* fB;
  double* C;                      // complex128, interleaved
  double* P;                      // nch > 1: FP64 partials [nch][Lt][Mp][Nc] complex
  int* Craw;                      // RAW mode: int32 [Mp][Brows]
  const int8_t* SA;               // tiled slices (tiled_off); RAW mode reads through the maps
  const int8_t* SB;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dev::smem_u32(dst)),
      "l"(map), "r"(dev::smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_64B: 8-row core-matrix groups 512 B apart
// (SBO), LBO unused for swizzled K-major, version 1 (sm_100), layout type 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}

// Slice layout of the Ozaki GEMM: tile-contiguous and pre-swizzled, [t][row block][k chunk]
// [slice][R rows][64 B], so one stage (all S slices of a k chunk) is one contiguous bulk copy
// (R = 128 for A, 64 for B).  Within a 64-byte row the 16-byte chunk index is XORed with
// (row >> 1) & 3: the SWIZZLE_64B pattern (byte-offset bits [4,6) ^= bits [7,9)) that TMA
// writes and UMMA reads.
template <int S, int R>
__device__ __forceinline__ size_t tiled_off(int t, int row, int kbyte, int nblk, int nk) {
  const int blk = row / R, r = row % R, kc = kbyte >> 6, c = kbyte & 63;
  return ((((size_t(t) * nblk + blk) * nk + kc) * S) * R + r) * 64 + ((((c >> 4) ^ ((r >> 1) & 3)) << 4) | (c & 15));
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dev::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(dev::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(dev::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// Splitting kernels

// x in (-1, 1) -> S signed slices (balanced base-256 digits) of m = round(x 2^F), F = 6 + 8 (S-1):
// from the least significant end, digit = low byte read as int8 (in [-128, 127]) and
// m = (m - digit) / 256 (exact); the top digit is what remains, |top| <= 2^6 + 1.  All slices
// are signed and zero-mean, so the truncated pair products (i + j >= S) and the rounding of x
// (|x - m 2^-F| <= 2^-F-1) add incoherently.  x 2^F is an exact power-of-two scaling.
template <int S>
__device__ __forceinline__ void split_value(double x, int8_t (&q)[S]) {
  constexpr int F = 6 + 8 * (S - 1);
  static_assert(F <= 62, "slices exceed int64");
  long long r = __double2ll_rn(x * static_cast<double>(1ll << F));
#pragma unroll
  for (int k = S - 1; k >= 1; --k) {
    const int dgt = int(int8_t(uint8_t(r & 255)));
    q[k] = int8_t(dgt);
    r = (r - dgt) >> 8;
  }
  q[0] = int8_t(r);
}

// 2^k for |k| <= 1000 (exact; the exponents here come from ilogb of finite data)
__device__ __forceinline__ double pow2(int k) {
  return __longlong_as_double(static_cast<long long>(1023 + k) << 52);
}

__device__ __forceinline__ int scale_exponent(double m) {
  // smallest e with m < 2^e (m > 0); 0 for an all-zero row / column
  return m > 0.0 ? ilogb(m) + 1 : 0;
}

// Operand addressing of a (two-level K) problem, complex elements (ZgemmProblem layout):
//   A(t, m, kk) = A + t sAb + (kk / Kin) sAo + m lda + kk % Kin
//   B(t, kk, n) = B + t sBb + (kk / Kin) sBo + (kk % Kin) ldb + n
// (K = Ko Kin < 2^31: 32-bit index arithmetic)
__device__ __forceinline__ const double2* a_at(const ZgemmProblem& q, int t, int64_t m, int kk) {
  if (q.Ko == 1) return static_cast<const double2*>(q.A) + t * q.sAb + m * q.lda + kk;
  const int ko = kk / int(q.Kin), ki = kk - ko * int(q.Kin);
  return static_cast<const double2*>(q.A) + t * q.sAb + ko * q.sAo + m * q.lda + ki;
}
__device__ __forceinline__ const double2* b_at(const ZgemmProblem& q, int t, int kk, int64_t n) {
  if (q.Ko == 1) return static_cast<const double2*>(q.B) + t * q.sBb + int64_t(kk) * q.ldb + n;
  const int ko = kk / int(q.Kin), ki = kk - ko * int(q.Kin);
  return static_cast<const double2*>(q.B) + t * q.sBb + ko * q.sBo + int64_t(ki) * q.ldb + n;
}

constexpr int KSEG = 4096;   // K elements per warp in the row kernels (long BB2 rows in parallel)
#ifndef SPLIT_COLS_ROWS
#define SPLIT_COLS_ROWS 32   // k rows per split_cols CTA (a multiple of 32; more CTAs for small N)
#endif

// Row scale exponents of A: grid (Mp/8, Lt, ceil(K/KSEG)), one warp per (row, K segment);
// eA preset to INT_MIN (bytes 0x80), segments folded in with atomicMax.
__global__ void __launch_bounds__(256) rowmax_kernel(ZgemmProblem q, int* __restrict__ eA, int Mp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = int64_t(blockIdx.x) * 8 + warp;
  const int t = blockIdx.y;
  if (i >= q.M) return;
  const int K = int(q.Kin * q.Ko);
  const int k0 = int(blockIdx.z) * KSEG, k1 = min(K, k0 + KSEG);
  double m = 0.0;
  for (int j = k0 + lane; j < k1; j += 32) {
    const double2 v = *a_at(q, t, i, j);
    m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0 && m > 0.0) atomicMax(&eA[size_t(t) * Mp + i], scale_exponent(m));
}

// A_cat row slices: grid (Mp/8, Lt, ceil(Kc/KSEG)), one warp per (row, K segment).  K index
// of A_cat: Re part of kk at kk, Im part at Kc + kk (Kc = roundup(K, 32)); padding rows /
// columns are zero; a row left at INT_MIN by rowmax_kernel is all zero (exponent 0).
template <int S>
__global__ void __launch_bounds__(256) split_rows_kernel(ZgemmProblem q, int8_t* __restrict__ SA,
                                                         const int* __restrict__ eA, int Mp, int Kc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = int64_t(blockIdx.x) * 8 + warp;
  const int t = blockIdx.y;
  if (i >= Mp) return;
  const int K = int(q.Kin * q.Ko);
  const bool live = i < q.M;
  const int Kp = 2 * Kc;
  const int nk = Kp / 64, nblk = Mp / 128;
  const int e0 = eA[size_t(t) * Mp + i];
  const double sc = pow2(e0 < -100000 ? 0 : -e0);
  const int j1 = min(Kc, int(blockIdx.z + 1) * KSEG);
  for (int j0 = int(blockIdx.z) * KSEG + lane * 4; j0 < j1; j0 += 128) {
    uint32_t wr[S], wi[S];
#pragma unroll
    for (int k = 0; k < S; ++k) wr[k] = wi[k] = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u;
      double2 v = make_double2(0.0, 0.0);
      if (live && j < K) v = *a_at(q, t, i, j);
      int8_t qr[S], qi[S];
      split_value<S>(v.x * sc, qr);
      split_value<S>(v.y * sc, qi);
#pragma unroll
      for (int k = 0; k < S; ++k) {
        wr[k] |= uint32_t(uint8_t(qr[k])) << (8 * u);
        wi[k] |= uint32_t(uint8_t(qi[k])) << (8 * u);
      }
    }
#pragma unroll
    for (int k = 0; k < S; ++k) {
      *reinterpret_cast<uint32_t*>(SA + tiled_off<S, 128>(t, int(i), j0, nblk, nk) + k * A_TILE) = wr[k];
      *reinterpret_cast<uint32_t*>(SA + tiled_off<S, 128>(t, int(i), Kc + j0, nblk, nk) + k * A_TILE) = wi[k];
    }
  }
}

// Column scale exponents of B: grid (Nc/32, Lt, ceil(K/128)); fB preset to INT_MIN (bytes 0x80),
// each CTA folds the max-exponent of its 128-row chunk in with atomicMax (exponents are
// monotone in the magnitude, so the max of the chunk exponents is the column's exponent).
__global__ void __launch_bounds__(256) colmax_kernel(ZgemmProblem q, int* __restrict__ fB, int Nc) {
  __shared__ double red[8][32];
  const int tid = threadIdx.x, c = tid & 31, r0 = tid >> 5;
  const int c0 = 32 * blockIdx.x, t = blockIdx.y;
  const int k0 = 128 * int(blockIdx.z), K = int(q.Kin * q.Ko);
  double m = 0.0;
  if (c0 + c < q.Nn) {
    const int k1 = min(K, k0 + 128);
    for (int k = k0 + r0; k < k1; k += 8) {
      const double2 v = *b_at(q, t, k, c0 + c);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
  }
  red[r0][c] = m;
  __syncthreads();
  if (tid < 32) {
#pragma unroll
    for (int r = 1; r < 8; ++r) m = fmax(m, red[r][tid]);
    m = fmax(m, red[0][tid]);
    if (m > 0.0 && c0 + tid < Nc) atomicMax(&fB[size_t(t) * Nc + c0 + tid], scale_exponent(m));
  }
}

// B_cat^T row slices: grid (Nc/CG, Lt, Kc/SPLIT_COLS_ROWS), one CTA per (CG-column group g, t,
// chunk of k rows).  A column left at INT_MIN by colmax_kernel is all zero (exponent 0).
template <int S, int BN>
__global__ void __launch_bounds__(256) split_cols_kernel(ZgemmProblem q, int8_t* __restrict__ SB,
                                                         const int* __restrict__ fB, int Nc, int Kc) {
  constexpr int CG = Tile<BN>::CG, B_TILE = Tile<BN>::B_TILE;
  __shared__ double2 tile[32][CG + 1];
  __shared__ int ecol[CG];
  const int tid = threadIdx.x;
  const int g = blockIdx.x, t = blockIdx.y;
  const int c0 = CG * g;
  const int K = int(q.Kin * q.Ko);
  const int Kp = 2 * Kc, Brows = 2 * Nc;
  const int nk = Kp / 64, nblk = Brows / BN;
  if (tid < CG) {
    const int e = fB[size_t(t) * Nc + c0 + tid];
    ecol[tid] = e < -100000 ? 0 : e;
  }
  const int kend = min(Kc, SPLIT_COLS_ROWS * int(blockIdx.z + 1));
  for (int k0 = SPLIT_COLS_ROWS * blockIdx.z; k0 < kend; k0 += 32) {
    __syncthreads();
    for (int idx = tid; idx < 32 * CG; idx += 256) {
      const int kr = idx / CG, c = idx % CG;
      double2 v = make_double2(0.0, 0.0);
      if (k0 + kr < K && c0 + c < q.Nn) v = *b_at(q, t, k0 + kr, c0 + c);
      tile[kr][c] = v;
    }
    __syncthreads();
    for (int item = tid; item < 16 * CG; item += 256) {
      const int kq = item & 3, h = (item >> 2) & 1, rT = item >> 3;
      const int c = rT % CG, part = rT / CG;
      const double sc = pow2(-ecol[c]);
      uint32_t lo[S], hi[S];
#pragma unroll
      for (int k = 0; k < S; ++k) lo[k] = hi[k] = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 v = tile[kq * 8 + u][c];
        // part 0 (Cr column): [Br; -Bi]; part 1 (Ci column): [Bi; Br]
        const double x = part == 0 ? (h == 0 ? v.x : -v.y) : (h == 0 ? v.y : v.x);
        int8_t qv[S];
        split_value<S>(x * sc, qv);
#pragma unroll
        for (int k = 0; k < S; ++k) {
          if (u < 4)
            lo[k] |= uint32_t(uint8_t(qv[k])) << (8 * u);
          else
            hi[k] |= uint32_t(uint8_t(qv[k])) << (8 * (u - 4));
        }
      }
#pragma unroll
      for (int k = 0; k < S; ++k)
        *reinterpret_cast<uint2*>(SB + tiled_off<S, BN>(t, BN * g + rT, h * Kc + k0 + kq * 8, nblk, nk) +
                                  k * B_TILE) = make_uint2(lo[k], hi[k]);
    }
  }
}

// Split-K reduction: C(t, m, n) = sum over chunks ch (in order) of P[ch][t][m][n].
__global__ void ozaki_reduce_kernel(Params p) {
  const int64_t total = int64_t(p.Lt) * p.M * p.Nn;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = e % p.Nn, m = (e / p.Nn) % p.M, t = e / (int64_t(p.Nn) * p.M);
    const double2* src = reinterpret_cast<const double2*>(p.P) + (t * p.Mp + m) * p.Nc + n;
    const int64_t stride = int64_t(p.Lt) * p.Mp * p.Nc;
    double2 acc = src[0];
    for (int ch = 1; ch < p.nch; ++ch) {
      const double2 v = src[ch * stride];
      acc.x += v.x;
      acc.y += v.y;
    }
    reinterpret_cast<double2*>(p.C)[t * p.sCb + m * p.ldc + n] = acc;
  }
}

// ---------------------------------------------------------------------------------------
// The tcgen05 GEMM, persistent: grid = min(tiles, SMs), 192 threads.
//   warps 0-3: epilogue (warp w drains TMEM lanes 32w..32w+31)
//   warp 4 lane 0: TMA producer, runs ahead across tiles through the stage ring
//   warp 5 lane 0: MMA issuer
// Tiles in (t, row block, column block) order, column blocks fastest (consecutive tiles of a
// CTA share the A slices in L2).  The S diagonal accumulators use S*64 of the 512 TMEM
// columns; the epilogue drains them in order d = 0..S-1 and releases each one (drained[d])
// as soon as it is in registers, so the next tile's MMAs into diagonal d start while the
// epilogue is still converting and storing.
template <int S, bool RAW, int BN>
__global__ void __launch_bounds__((Tile<BN>::NEPI + 2) * 32, 1) ozaki_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                                                            const __grid_constant__ CUtensorMap mapB, Params p) {
  using C = Cfg<S, BN>;
  constexpr int CG = Tile<BN>::CG, NEPI = Tile<BN>::NEPI, CPW = Tile<BN>::CPW, B_TILE = Tile<BN>::B_TILE;
  constexpr uint32_t IDESC = Tile<BN>::IDESC;
  extern __shared__ __align__(1024) uint8_t dsm[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES], tfull, drained[S];
  __shared__ uint32_t tmem_slot;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = p.Brows / BN, ntm = p.Mp / BM;
  const int ntiles = ntn * ntm * (RAW ? 1 : p.Lt) * p.nch;   // (t, row block, column block, K chunk)

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dev::smem_u32(&tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < C::STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    dev::mbar_init(&tfull, 1);
    for (int d = 0; d < S; ++d) dev::mbar_init(&drained[d], NEPI);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int nk = p.Kp / BKB;
  // tile -> (t, mb, nb, ch), K chunks fastest; chunk ch covers stages [ch kchs, kc1)
  auto decode = [&](int tile, int& t, int& mb, int& nb, int& ch) {
    ch = tile % p.nch;
    const int r = tile / p.nch;
    nb = r % ntn;
    mb = (r / ntn) % ntm;
    t = r / (ntn * ntm);
  };

  if (warp == NEPI) {
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int t, mb, nb, ch;
        decode(tile, t, mb, nb, ch);
        const int rowA = t * p.Mp + mb * BM;
        const int rowB = t * p.Brows + nb * BN;
        const int kc1 = min(nk, (ch + 1) * p.kchs);
        for (int kc = ch * p.kchs; kc < kc1; ++kc, ++it) {
          const int st = it % C::STAGES;
          if (it >= C::STAGES) dev::mbar_wait(&empty[st], ((it / C::STAGES) - 1) & 1);
          dev::mbar_expect_tx(&full[st], C::STAGE);
          uint8_t* sa = smem + st * C::STAGE;
          uint8_t* sb = sa + S * A_TILE;
          if constexpr (RAW) {
            tma_load_2d(sa, &mapA, &full[st], kc * BKB, rowA);
            tma_load_2d(sb, &mapB, &full[st], kc * BKB, rowB);
          } else {
            bulk_load(sa, p.SA + ((size_t(t) * ntm + mb) * nk + kc) * (S * A_TILE), S * A_TILE, &full[st]);
            bulk_load(sb, p.SB + ((size_t(t) * ntn + nb) * nk + kc) * (S * B_TILE), S * B_TILE, &full[st]);
          }
        }
      }
    }
  } else if (warp == NEPI + 1) {
    if (lane == 0) {
      int it = 0, n = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++n) {
        const int ch = tile % p.nch;
        const int kc0 = ch * p.kchs, kc1 = min(nk, (ch + 1) * p.kchs);
        for (int kc = kc0; kc < kc1; ++kc, ++it) {
          const int st = it % C::STAGES;
          dev::mbar_wait(&full[st], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = dev::smem_u32(smem + st * C::STAGE);
          const uint32_t sb = sa + S * A_TILE;
#pragma unroll
          for (int d = 0; d < S; ++d) {
            if (kc == kc0 && n > 0) {
              dev::mbar_wait(&drained[d], (n - 1) & 1);     // previous tile's diagonal d is in registers
              tc_fence_after();
            }
#pragma unroll
            for (int i = 0; i <= d; ++i)
#pragma unroll
              for (int ks = 0; ks < BKB / UK; ++ks)
                mma_i8(tmem + uint32_t(d * BN), sw64_desc(sa + i * A_TILE + ks * UK),
                       sw64_desc(sb + (d - i) * B_TILE + ks * UK), IDESC, ((kc - kc0) | i | ks) != 0);
          }
          mma_commit(&empty[st]);
        }
        mma_commit(&tfull);
      }
    }
  } else {
    int n = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++n) {
      int t, mb, nb, ch;
      decode(tile, t, mb, nb, ch);
      dev::mbar_wait(&tfull, n & 1);
      tc_fence_after();
      const int quarter = warp & 3, half = warp >> 2;            // TMEM lane quarter, column half
      const int r = mb * BM + quarter * 32 + lane;                // row of this thread (TMEM lane)
      const uint32_t tl = tmem + (uint32_t(quarter * 32) << 16);
      if constexpr (RAW) {
        if (half == 0) {
#pragma unroll
          for (int q = 0; q < BN / 16; ++q) {
            int v[16];
            tmem_ld16(tl + q * 16, v);
            tmem_wait_ld();
            if (q == BN / 16 - 1) tc_fence_before();
            int* dst = p.Craw + size_t(r) * p.Brows + nb * BN + q * 16;
#pragma unroll
            for (int u = 0; u < 16; u += 4)
              *reinterpret_cast<int4*>(dst + u) = make_int4(v[u], v[u + 1], v[u + 2], v[u + 3]);
          }
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&drained[0]);
      } else {
        double ar[CPW], ai[CPW];
#pragma unroll
        for (int q = 0; q < CPW; ++q) ar[q] = ai[q] = 0.0;
#pragma unroll 1
        for (int d = 0; d < S; ++d) {          // most significant accumulator first (fixed order)
          int vr[CPW], vi[CPW];
#pragma unroll
          for (int q = 0; q < CPW; q += 8) {
            tmem_ld8(tl + uint32_t(d * BN + half * CPW + q), &vr[q]);
            tmem_ld8(tl + uint32_t(d * BN + CG + half * CPW + q), &vi[q]);
          }
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) dev::mbar_arrive(&drained[d]);
          const double w = pow2(-12 - 8 * d);
#pragma unroll
          for (int q = 0; q < CPW; ++q) {
            ar[q] = fma(double(vr[q]), w, ar[q]);
            ai[q] = fma(double(vi[q]), w, ai[q]);
          }
        }
        if (r < p.M) {
          const int ea = p.eA[size_t(t) * p.Mp + r];
          const double se = pow2(ea < -100000 ? 0 : ea);        // INT_MIN: an all-zero row
          const int cbase = nb * CG + half * CPW;
          const int* f = p.fB + size_t(t) * p.Nc + cbase;
          // one K chunk: the tile itself; else this chunk's FP64 partial (reduced in order later)
          double* dst = p.nch == 1 ? p.C + 2 * (size_t(t) * p.sCb + size_t(r) * p.ldc)
                                   : p.P + 2 * (((size_t(ch) * p.Lt + t) * p.Mp + r) * p.Nc);
#pragma unroll
          for (int q = 0; q < CPW; ++q) {
            const int c = cbase + q;
            if (c < p.Nn) {
              const double sf = se * pow2(f[q] < -100000 ? 0 : f[q]);   // exact: a power of two
              *reinterpret_cast<double2*>(dst + 2 * c) = make_double2(ar[q] * sf, ai[q] * sf);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(q);
  });
  return fn;
}

bool map_i8(CUtensorMap* map, const void* base, uint64_t kp, uint64_t rows, uint32_t box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t gd[2] = {kp, rows};
  cuuint64_t gs[1] = {kp};
  cuuint32_t box[2] = {uint32_t(BKB), box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), gd, gs, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Sizes of one problem's slices for a batch of Lt time slices.
struct Geometry {
  int Mp, Nc, Kc, Kp, Brows, nk, kchs, nch;
  size_t sa, ea, sb, fb, part, total;   // offsets in the workspace: A slices, eA, B slices, fB, partials
  size_t a_form() const { return (ea - sa) + (sb - ea); }     // A slices + eA
  size_t b_form() const { return (fb - sb) + (part - fb); }   // B slices + fB
};

constexpr int KCH_BYTES = 16384;   // K bytes per chunk: |acc| <= 7 * 2^14 * 16384 < 2^31

// Tile width for a problem: 96 when the output is wide enough that padding to 48 columns
// costs <= 3 % and the S accumulators fit TMEM (S <= 5), else 64.
int pick_bn(const ZgemmProblem& q, int S) { return q.Nn >= 512 && S * 96 <= 512 ? 96 : 64; }

Geometry geometry(const ZgemmProblem& q, int64_t Lt, int S, int BN) {
  Geometry g;
  const int64_t K = q.Kin * q.Ko;
  g.Mp = int((q.M + BM - 1) / BM * BM);
  g.Nc = int((q.Nn + BN / 2 - 1) / (BN / 2) * (BN / 2));
  g.Kc = int((K + 31) / 32 * 32);
  g.Kp = 2 * g.Kc;
  g.Brows = 2 * g.Nc;
  g.nk = g.Kp / BKB;
  g.kchs = std::min(g.nk, KCH_BYTES / BKB);
  g.nch = (g.nk + g.kchs - 1) / g.kchs;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  g.sa = 0;
  g.ea = al(size_t(S) * Lt * g.Mp * g.Kp);
  g.sb = g.ea + al(size_t(Lt) * g.Mp * 4);
  g.fb = g.sb + al(size_t(S) * Lt * g.Brows * g.Kp);
  g.part = g.fb + al(size_t(Lt) * g.Nc * 4);
  g.total = g.part + (g.nch > 1 ? al(size_t(g.nch) * Lt * g.Mp * g.Nc * 16) : 0);
  return g;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int S, bool RAW, int BN>
cudaError_t launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t stream) {
  using C = Cfg<S, BN>;
  auto k = ozaki_gemm_kernel<S, RAW, BN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles = int64_t(p.Brows / BN) * (p.Mp / BM) * (RAW ? 1 : p.Lt) * p.nch;
  const int grid = int(tiles < num_sms() ? tiles : num_sms());
  k<<<grid, (Tile<BN>::NEPI + 2) * 32, C::SMEM, stream>>>(ma, mb, p);
  return cudaGetLastError();
}

template <int S>
cudaError_t split_a(const ZgemmProblem& q, int8_t* SA, int* eA, const Geometry& g, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(eA, 0x80, size_t(q.batch) * g.Mp * 4, stream);   // INT_MIN-like
  if (e != cudaSuccess) return e;
  const int64_t K = q.Kin * q.Ko;
  rowmax_kernel<<<dim3(g.Mp / 8, unsigned(q.batch), unsigned((K + KSEG - 1) / KSEG)), 256, 0, stream>>>(q, eA, g.Mp);
  split_rows_kernel<S><<<dim3(g.Mp / 8, unsigned(q.batch), unsigned((g.Kc + KSEG - 1) / KSEG)), 256, 0, stream>>>(
      q, SA, eA, g.Mp, g.Kc);
  return cudaGetLastError();
}

template <int S, int BN>
cudaError_t split_b(const ZgemmProblem& q, int8_t* SB, int* fB, const Geometry& g, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(fB, 0x80, size_t(q.batch) * g.Nc * 4, stream);   // INT_MIN-like
  if (e != cudaSuccess) return e;
  const int64_t K = q.Kin * q.Ko;
  colmax_kernel<<<dim3((g.Nc + 31) / 32, unsigned(q.batch), unsigned((K + 127) / 128)), 256, 0, stream>>>(q, fB, g.Nc);
  split_cols_kernel<S, BN><<<dim3(g.Nc / Tile<BN>::CG, unsigned(q.batch), unsigned((g.Kc + SPLIT_COLS_ROWS - 1) / SPLIT_COLS_ROWS)), 256, 0, stream>>>(q, SB, fB,
                                                                                                          g.Nc, g.Kc);
  return cudaGetLastError();
}

// One batch (q.batch time slices): split what is not pre-split, GEMM, split-K reduction.
template <int S, int BN>
cudaError_t run_batch(const ZgemmProblem& q, uint8_t* w, const OzakiForm* fa, const OzakiForm* fb,
                      cudaStream_t stream) {
  const Geometry g = geometry(q, q.batch, S, BN);
  const int8_t* SA = reinterpret_cast<int8_t*>(w + g.sa);
  const int* eA = reinterpret_cast<int*>(w + g.ea);
  const int8_t* SB = reinterpret_cast<int8_t*>(w + g.sb);
  const int* fB = reinterpret_cast<int*>(w + g.fb);
  if (fa) {
    SA = static_cast<const int8_t*>(fa->slices);
    eA = fa->exps;
  } else {
    cudaError_t e = split_a<S>(q, reinterpret_cast<int8_t*>(w + g.sa), reinterpret_cast<int*>(w + g.ea), g, stream);
    if (e != cudaSuccess) return e;
  }
  if (fb) {
    SB = static_cast<const int8_t*>(fb->slices);
    fB = fb->exps;
  } else {
    cudaError_t e = split_b<S, BN>(q, reinterpret_cast<int8_t*>(w + g.sb), reinterpret_cast<int*>(w + g.fb), g, stream);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap ma{}, mb{};   // unused: the slices are tile-contiguous, read by bulk copies
  Params p{};
  p.Lt = int(q.batch); p.Mp = g.Mp; p.Nc = g.Nc; p.Kp = g.Kp; p.Brows = g.Brows;
  p.M = int(q.M); p.Nn = int(q.Nn); p.nch = g.nch; p.kchs = g.kchs;
  p.ldc = q.ldc; p.sCb = q.sCb;
  p.eA = eA; p.fB = fB; p.C = static_cast<double*>(q.C);
  p.P = g.nch > 1 ? reinterpret_cast<double*>(w + g.part) : nullptr;
  p.SA = SA; p.SB = SB;
  e = launch_gemm<S, false, BN>(ma, mb, p, stream);
  if (e != cudaSuccess || g.nch == 1) return e;
  ozaki_reduce_kernel<<<num_sms() * 4, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

// The whole problem in batches of time slices that fit the workspace (pre-split forms only
// when it fits in one batch).
template <int S, int BN>
cudaError_t run_gemm(const ZgemmProblem& q, void* ws, size_t ws_bytes, const OzakiForm* fa, const OzakiForm* fb,
                     cudaStream_t stream) {
  int64_t bt = q.batch;
  while (bt > 1 && geometry(q, bt, S, BN).total > ws_bytes) bt = (bt + 1) / 2;
  if (geometry(q, bt, S, BN).total > ws_bytes) return cudaErrorInvalidValue;
  if (bt < q.batch) fa = fb = nullptr;
  for (int64_t t0 = 0; t0 < q.batch; t0 += bt) {
    ZgemmProblem b = q;
    b.batch = std::min(bt, q.batch - t0);
    b.A = static_cast<const double2*>(q.A) + t0 * q.sAb;
    b.B = static_cast<const double2*>(q.B) + t0 * q.sBb;
    b.C = static_cast<double2*>(q.C) + t0 * q.sCb;
    cudaError_t e = run_batch<S, BN>(b, static_cast<uint8_t*>(ws), fa, fb, stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int S, int BN>
cudaError_t make_form(const ZgemmProblem& q, bool as_b, void* dst, OzakiForm* form, cudaStream_t stream) {
  const Geometry g = geometry(q, q.batch, S, BN);
  uint8_t* d = static_cast<uint8_t*>(dst);
  form->slices = d;
  if (!as_b) {
    form->exps = reinterpret_cast<const int*>(d + (g.ea - g.sa));
    return split_a<S>(q, reinterpret_cast<int8_t*>(d), reinterpret_cast<int*>(d + (g.ea - g.sa)), g, stream);
  }
  form->exps = reinterpret_cast<const int*>(d + (g.fb - g.sb));
  return split_b<S, BN>(q, reinterpret_cast<int8_t*>(d), reinterpret_cast<int*>(d + (g.fb - g.sb)), g, stream);
}

ZgemmProblem mm1_problem(const void* A, const void* B, void* C, int64_t Lt, int64_t N) {
  ZgemmProblem q{};
  q.A = A; q.B = B; q.C = C; q.batch = Lt;
  q.M = N; q.Nn = N; q.Kin = N; q.Ko = 1;
  q.lda = N; q.sAo = 0; q.sAb = N * N;
  q.ldb = N; q.sBo = 0; q.sBb = N * N;
  q.ldc = N; q.sCb = N * N;
  return q;
}

}  // namespace oz

// slice counts whose S diagonal accumulators fit the 512 TMEM columns at the problem's tile width
#define OZ_CASE(k, bn, fn, ...) \
  case k:                       \
    if constexpr (k * bn <= 512) return oz::fn<k, bn>(__VA_ARGS__); else return cudaErrorInvalidValue;
#define OZ_SWITCH(bn, fn, ...)                  \
  switch (slices) {                             \
    OZ_CASE(4, bn, fn, __VA_ARGS__)             \
    OZ_CASE(5, bn, fn, __VA_ARGS__)             \
    OZ_CASE(6, bn, fn, __VA_ARGS__)             \
    OZ_CASE(7, bn, fn, __VA_ARGS__)             \
    default: return cudaErrorInvalidValue;      \
  }
#define OZ_DISPATCH(q, fn, ...)                                   \
  if (oz::pick_bn(q, slices) == 96) { OZ_SWITCH(96, fn, __VA_ARGS__) }    \
  else { OZ_SWITCH(64, fn, __VA_ARGS__) }

size_t ozaki_workspace_bytes(const ZgemmProblem& q, int slices, int64_t max_batch) {
  return oz::geometry(q, std::max<int64_t>(1, std::min(max_batch, q.batch)), slices, oz::pick_bn(q, slices)).total;
}
size_t ozaki_mm1_workspace_bytes(int64_t Lt, int64_t N, int slices) {
  return ozaki_workspace_bytes(oz::mm1_problem(nullptr, nullptr, nullptr, Lt, N), slices, Lt);
}
size_t ozaki_form_bytes(const ZgemmProblem& q, int slices, bool as_b) {
  const oz::Geometry g = oz::geometry(q, q.batch, slices, oz::pick_bn(q, slices));
  return as_b ? g.b_form() : g.a_form();
}
cudaError_t launch_ozaki_form(const ZgemmProblem& q, int slices, bool as_b, void* dst, OzakiForm* form,
                              cudaStream_t stream) {
  OZ_DISPATCH(q, make_form, q, as_b, dst, form, stream)
}
cudaError_t launch_ozaki_gemm(const ZgemmProblem& q, int slices, void* ws, size_t ws_bytes, cudaStream_t stream,
                              const OzakiForm* fa, const OzakiForm* fb) {
  OZ_DISPATCH(q, run_gemm, q, ws, ws_bytes, fa, fb, stream)
}
cudaError_t launch_ozaki_mm1(const void* A, const void* B, void* C, int64_t Lt, int64_t N, int slices, void* ws,
                             size_t ws_bytes, cudaStream_t stream, const OzakiForm* fa, const OzakiForm* fb) {
  return launch_ozaki_gemm(oz::mm1_problem(A, B, C, Lt, N), slices, ws, ws_bytes, stream, fa, fb);
}

cudaError_t launch_i8gemm_tn(const int8_t* A, const int8_t* B, int32_t* C, int64_t M, int64_t Nn, int64_t K,
                             cudaStream_t stream) {
  // tile width 96 when M % 256 == 0, else 64 (both widths pinned by the bit-exact tests)
  const int bn = (M % 256 == 0 && Nn % 96 == 0) ? 96 : 64;
  if (M % oz::BM || Nn % bn || K % oz::BKB) return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  if (!oz::map_i8(&ma, A, uint64_t(K), uint64_t(M), oz::BM) || !oz::map_i8(&mb, B, uint64_t(K), uint64_t(Nn), uint32_t(bn)))
    return cudaErrorInvalidValue;
  oz::Params p{};
  p.Lt = 1; p.Mp = int(M); p.Nc = int(Nn / 2); p.Kp = int(K); p.Brows = int(Nn);
  p.M = int(M); p.Nn = int(Nn); p.nch = 1; p.kchs = int(K / oz::BKB);
  p.Craw = C;
  return bn == 96 ? oz::launch_gemm<1, true, 96>(ma, mb, p, stream) : oz::launch_gemm<1, true, 64>(ma, mb, p, stream);
}

}  // namespace cc
