// Device helpers shared by the contraction kernels (sm_100a): mbarrier, TMA, FP64 DMMA,
// acquire/release, the DMMA tile configuration and the complex DMMA k-tile step.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace cc {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// sign flip as an integer XOR on the high word (ALU pipe, not the FP64 pipe)
__device__ __forceinline__ double neg(double x) {
  double r;
  asm("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %1;\nxor.b32 hi, hi, 0x80000000;\nmov.b64 %0, {lo, hi};\n}" : "=d"(r) : "d"(x));
  return r;
}

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NCW = WARPS_M * WARPS_N;  // consumer (DMMA) warps
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int MI = WM / 8, NI = WN / 4;
  static constexpr int NJ = WN / 8;              // 3M: 8-complex column blocks per warp tile
  static constexpr int FRAG = MI * NI * 2;       // accumulator doubles per lane
  static constexpr int A_BYTES = BM * BK * 16, B_BYTES = BK * BN * 16;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 1024;
  static constexpr int SLOT_DOUBLES = NCW * FRAG * 32;
  static_assert(BK % 8 == 0 && BN % 8 == 0 && BM % 8 == 0, "tile dims");
  static_assert(WM % 8 == 0 && WN % 4 == 0, "warp tile dims");
  static_assert((BM * 128) % 1024 == 0 && (BK * 128) % 1024 == 0, "128B swizzle needs 1024B-aligned sub-tiles");
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// One k-tile (BK complex) of a warp's WM x WN complex accumulator block from the stage's
// swizzled shared-memory tiles (see zgemm.cu header for the fragment mapping).  Lane
// (g = lane/4, t = lane%4); rows of the warp start at row0 = wm*WM, its complex columns at
// col0 = wn*WN.  With WM, WN multiples of 8 every swizzle key is a lane constant:
// A row r = row0 + 8i + g has key g; B column n = col0 + 4k + g/2 sits in 128-byte chunk
// n/8 = col0/8 + k/2 at slot 4(k%2) + g/2.
template <class C>
__device__ __forceinline__ void dmma_ktile(const uint8_t* sA, const uint8_t* sB, int wm, int wn, int g, int t,
                                           bool q, double (&acc)[C::MI][C::NI][2]) {
  static_assert(C::WM % 8 == 0 && C::WN % 8 == 0, "lane-constant swizzle keys need WM, WN % 8 == 0");
  const uint8_t* a_base = sA + (wm * C::WM + g) * 128;
  const uint8_t* b_base = sB + (wn * C::WN / 8) * (C::BK * 128);
#pragma unroll
  for (int kc = 0; kc < C::BK / 8; ++kc) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * t + h;       // complex k slot within the 8-complex chunk
      const int krow = kc * 8 + s;   // B row within the stage (krow & 7 == s)
      double2 a[C::MI];
      double b_re_row[C::NI], b_im_row[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
        a[i] = *reinterpret_cast<const double2*>(a_base + kc * C::BM * 128 + i * 1024 + ((s ^ g) << 4));
#pragma unroll
      for (int k = 0; k < C::NI; ++k) {
        const int slot = 4 * (k & 1) + (g >> 1);
        const double2 bv = *reinterpret_cast<const double2*>(b_base + (k >> 1) * (C::BK * 128) + krow * 128 +
                                                             ((slot ^ s) << 4));
        // B' = [[br, bi], [-bi, br]]: row (k, re) -> (br | bi), row (k, im) -> (-bi | br)
        b_re_row[k] = q ? bv.y : bv.x;
        b_im_row[k] = q ? bv.x : neg(bv.y);
      }
      // two sweeps: dependent DMMAs on one accumulator are MI*NI instructions apart
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int k = 0; k < C::NI; ++k) dmma(acc[i][k][0], acc[i][k][1], a[i].x, b_re_row[k]);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int k = 0; k < C::NI; ++k) dmma(acc[i][k][0], acc[i][k][1], a[i].y, b_im_row[k]);
    }
  }
}

// 3M (Gauss) form of the same k-tile: three real products per complex one,
//   P0 += Ar Br,  P1 += Ai Bi,  P2 += (Ar + Ai)(Br + Bi),
// so that C = (P0 - P1) + i (P2 - P0 - P1) (see gauss3m_combine): 6 instead of 8 real flops
// per complex MAC (reading V-3).  The DMMA k index t of lane (g, t) is complex
// k = 8 kc + 2t + h for both operands (same conflict-free permutation as dmma_ktile); the
// real accumulator D[g][2t + e] of block (i, j) is complex C[row0 + 8i + g][col0 + 8j + 2t + e].
// The operand sums of one k-quad as ONE asm block: the FP64 adds share the datapath with the
// DMMAs, and grouping them keeps the compiler from scattering them between DMMAs.
template <int MI, int NJ>
__device__ __forceinline__ void gauss3m_sums(const double (&ar)[MI], const double (&ai)[MI], double (&as)[MI],
                                             const double (&br)[NJ], const double (&bi)[NJ], double (&bs)[NJ]) {
  static_assert(MI == 4 && NJ == 2, "grouped sums are written for the 32 x 16 warp tile");
  asm("add.f64 %0, %6, %7;\n\tadd.f64 %1, %8, %9;\n\tadd.f64 %2, %10, %11;\n\tadd.f64 %3, %12, %13;\n\t"
      "add.f64 %4, %14, %15;\n\tadd.f64 %5, %16, %17;"
      : "=d"(as[0]), "=d"(as[1]), "=d"(as[2]), "=d"(as[3]), "=d"(bs[0]), "=d"(bs[1])
      : "d"(ar[0]), "d"(ai[0]), "d"(ar[1]), "d"(ai[1]), "d"(ar[2]), "d"(ai[2]), "d"(ar[3]), "d"(ai[3]), "d"(br[0]),
        "d"(bi[0]), "d"(br[1]), "d"(bi[1]));
}

// `between(q)` runs after the DMMA sweeps of k-quad q (0..BK/4-1): other work (the dataflow
// worker's interleaved trace rows) issued while this warp's DMMAs drain from the FP64 pipe.
template <class C, class F>
__device__ __forceinline__ void dmma3m_ktile(const uint8_t* sA, const uint8_t* sB, int wm, int wn, int g, int t,
                                             double (&p)[3][C::MI][C::NJ][2], F&& between) {
  static_assert(C::WM % 8 == 0 && C::WN % 8 == 0, "lane-constant swizzle keys need WM, WN % 8 == 0");
  const uint8_t* a_base = sA + (wm * C::WM + g) * 128;
  const uint8_t* b_base = sB + (wn * C::WN / 8) * (C::BK * 128);
#pragma unroll
  for (int kc = 0; kc < C::BK / 8; ++kc) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * t + h;       // complex k slot within the 8-complex chunk
      const int krow = kc * 8 + s;   // B row within the stage (krow & 7 == s)
      double ar[C::MI], ai[C::MI], as[C::MI], br[C::NJ], bi[C::NJ], bs[C::NJ];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const double2 a = *reinterpret_cast<const double2*>(a_base + kc * C::BM * 128 + i * 1024 + ((s ^ g) << 4));
        ar[i] = a.x;
        ai[i] = a.y;
      }
#pragma unroll
      for (int j = 0; j < C::NJ; ++j) {
        const double2 b = *reinterpret_cast<const double2*>(b_base + j * (C::BK * 128) + krow * 128 + ((g ^ s) << 4));
        br[j] = b.x;
        bi[j] = b.y;
      }
      gauss3m_sums<C::MI, C::NJ>(ar, ai, as, br, bi, bs);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NJ; ++j) dmma(p[0][i][j][0], p[0][i][j][1], ar[i], br[j]);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NJ; ++j) dmma(p[1][i][j][0], p[1][i][j][1], ai[i], bi[j]);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NJ; ++j) dmma(p[2][i][j][0], p[2][i][j][1], as[i], bs[j]);
      between(2 * kc + h);
    }
  }
}
template <class C>
__device__ __forceinline__ void dmma3m_ktile(const uint8_t* sA, const uint8_t* sB, int wm, int wn, int g, int t,
                                             double (&p)[3][C::MI][C::NJ][2]) {
  dmma3m_ktile<C>(sA, sB, wm, wn, g, t, p, [](int) {});
}
// complex result of the 3M products of accumulator (i, j, e)
template <class C>
__device__ __forceinline__ double2 gauss3m_combine(const double (&p)[3][C::MI][C::NJ][2], int i, int j, int e) {
  return make_double2(p[0][i][j][e] - p[1][i][j][e], (p[2][i][j][e] - p[0][i][j][e]) - p[1][i][j][e]);
}

using Big = Cfg<64, 64, 16, 32, 16, 4>;

}  // namespace dev
}  // namespace cc
