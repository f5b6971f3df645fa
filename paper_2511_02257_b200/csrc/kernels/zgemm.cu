// Batched complex-double GEMM on FP64 DMMA tensor cores, fed by TMA (sm_100a).
//
// Serves the three "exterior contract" kinds (index semantics DESIGN.md
// reading V-1): MM1 (meson x meson, O(N^3)), BM1 (baryon x meson, single
// index, O(N^4)) and BB2 (baryon x baryon, double index + spin, O(N^4)) are
// one batched GEMM with a two-level K index after index fusion (kernels.hpp).
//
// Design:
//  - complex arithmetic as the real embedding: A is read as real [M][2K] (interleaved
//    complex already is), B is expanded on the fly into 2x2 blocks [[br, bi], [-bi, br]],
//    C comes out interleaved; one real GEMM, 8 real flops per complex MAC (4M, V-3).
//  - FP64 tensor cores: mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4 (tcgen05 has no f64 kind).
//    A warp tile of WM rows x WN complex columns keeps (WM/8)*(WN/4) accumulator pairs.
//  - K-slot permutation: lane t of an 8x4 fragment holds complex k = 2t+h (h = 0,1) of an
//    8-complex chunk, re part for the first DMMA and im part for the second, so each lane
//    does one 16-byte shared load per operand per (chunk, h) and both loads are free of
//    bank conflicts under the TMA 128-byte swizzle.
//  - TMA (cp.async.bulk.tensor, SWIZZLE_128B, zero fill out of bounds for ragged tails),
//    STAGES-deep mbarrier ring, one producer warp, NCW consumer warps.
//  - persistent stream-K: grid = #SMs, CTA c owns the contiguous k-iteration range
//    [c*T/G, (c+1)*T/G) of the flattened (tile, k-tile) space, so every SM gets the same
//    number of DMMA k-iterations (no wave quantisation) and the TMA ring streams across tile
//    boundaries.  A tile split between CTAs is finished by the CTA holding its last
//    k-iteration ("owner"), which adds the partials of the earlier CTAs in a fixed order
//    (c-1, c-2, ...), read from an L2 workspace after a per-warp release/acquire flag; every
//    CTA first computes the head of its last, shared tile so owners never wait long.
//    No floating-point atomics: results are bit-identical run to run.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "kernels.hpp"

namespace cc {
namespace {
using namespace dev;

struct KArgs {
  double2* C;
  double* ws;           // G slots x NCW warps x (MI*NI*2) x 32 lanes doubles
  int* flags;           // G x NCW; zero on entry and on exit
  int64_t M, Nn, ldc, sCb;
  int64_t total;        // n_tiles * KT
  int32_t tiles_m, tiles_n, kt_per_o, KT, G;
};

// The k-iteration range of CTA c and its segments (one per tile touched), in processing
// order: the head of a shared last tile first, then the tiles in ascending order.
struct Range {
  int64_t s, e;
  int64_t first_tile, last_tile;
  bool reorder;
  __device__ Range(const KArgs& a, int c) {
    s = (int64_t(c) * a.total) / a.G;
    e = (int64_t(c + 1) * a.total) / a.G;
    first_tile = s / a.KT;
    last_tile = (e - 1) / a.KT;
    reorder = (last_tile > first_tile) && (e - last_tile * a.KT < a.KT);
  }
  __device__ int64_t count() const { return e > s ? last_tile - first_tile + 1 : 0; }
  __device__ int64_t tile(int64_t j) const {
    if (!reorder) return first_tile + j;
    return j == 0 ? last_tile : first_tile + j - 1;
  }
};

__device__ __forceinline__ int64_t range_start(int64_t c, const KArgs& a) { return (c * a.total) / a.G; }

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
    zgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, KArgs args) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned stage base, derived from the __shared__ array by pointer arithmetic so
  // the compiler keeps the shared address space (LDS, not generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const Range rg(args, cta);
  const int64_t n_seg = rg.count();
  const int64_t tiles_mn = int64_t(args.tiles_m) * args.tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == C::NCW) {
    // ----------------------------- TMA producer ---------------------------------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t j = 0; j < n_seg; ++j) {
        const int64_t tile = rg.tile(j);
        const int64_t b = tile / tiles_mn;
        const int64_t r = tile - b * tiles_mn;
        const int tn = int(r / args.tiles_m), tm = int(r - int64_t(tn) * args.tiles_m);
        const int64_t base = tile * args.KT;
        const int k0 = int((rg.s > base ? rg.s : base) - base);
        const int k1 = int((rg.e < base + args.KT ? rg.e : base + args.KT) - base);
        for (int k = k0; k < k1; ++k) {
          const int ko = k / args.kt_per_o;
          const int ki0 = (k - ko * args.kt_per_o) * C::BK;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* sA = smem + stage * C::STAGE_BYTES;
          uint8_t* sB = sA + C::A_BYTES;
#pragma unroll
          for (int kc = 0; kc < C::BK / 8; ++kc)
            tma_load_4d(sA + kc * C::BM * 128, &tmA, &full[stage], 2 * (ki0 + kc * 8), tm * C::BM, ko, int(b));
#pragma unroll
          for (int nc = 0; nc < C::BN / 8; ++nc)
            tma_load_4d(sB + nc * C::BK * 128, &tmB, &full[stage], 2 * (tn * C::BN + nc * 8), ki0, ko, int(b));
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ------------------------------- DMMA consumers -------------------------------------
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int g = lane >> 2, t = lane & 3;
  const bool q = (g & 1) != 0;  // real column parity of this lane's B fragment column
  int a_row_off[C::MI], a_key[C::MI];
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    const int r = wm * C::WM + i * 8 + g;
    a_row_off[i] = r * 128;
    a_key[i] = r & 7;
  }
  int b_col_off[C::NI], b_slot[C::NI];
#pragma unroll
  for (int k = 0; k < C::NI; ++k) {
    const int n = wn * C::WN + k * 4 + (g >> 1);
    b_col_off[k] = (n >> 3) * C::BK * 128;
    b_slot[k] = n & 7;
  }

  int stage = 0;
  uint32_t phase = 0;
  for (int64_t j = 0; j < n_seg; ++j) {
    const int64_t tile = rg.tile(j);
    const int64_t base = tile * args.KT;
    const int k0 = int((rg.s > base ? rg.s : base) - base);
    const int k1 = int((rg.e < base + args.KT ? rg.e : base + args.KT) - base);
    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int k = 0; k < C::NI; ++k) acc[i][k][0] = acc[i][k][1] = 0.0;

    for (int kk = k0; kk < k1; ++kk) {
      mbar_wait(&full[stage], phase);
      const uint8_t* sA = smem + stage * C::STAGE_BYTES;
      const uint8_t* sB = sA + C::A_BYTES;
#pragma unroll
      for (int kc = 0; kc < C::BK / 8; ++kc) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int s = 2 * t + h;       // complex k slot within the 8-complex chunk
          const int krow = kc * 8 + s;   // B row within the stage
          double2 a[C::MI];
#pragma unroll
          for (int i = 0; i < C::MI; ++i)
            a[i] = *reinterpret_cast<const double2*>(sA + kc * C::BM * 128 + a_row_off[i] + ((s ^ a_key[i]) << 4));
#pragma unroll
          for (int k = 0; k < C::NI; ++k) {
            const double2 bv =
                *reinterpret_cast<const double2*>(sB + b_col_off[k] + krow * 128 + ((b_slot[k] ^ (krow & 7)) << 4));
            // B' = [[br, bi], [-bi, br]]: row (k, re) -> (br | bi), row (k, im) -> (-bi | br)
            const double b_re_row = q ? bv.y : bv.x;
            const double b_im_row = q ? bv.x : neg(bv.y);
#pragma unroll
            for (int i = 0; i < C::MI; ++i) {
              dmma(acc[i][k][0], acc[i][k][1], a[i].x, b_re_row);
              dmma(acc[i][k][0], acc[i][k][1], a[i].y, b_im_row);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    if (k1 < args.KT) {
      // contributor: publish this warp's partial fragment for the tile's owner
      double* slot = args.ws + (int64_t(cta) * C::NCW + warp) * (C::FRAG * 32);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int k = 0; k < C::NI; ++k) {
          __stcg(slot + ((i * C::NI + k) * 2 + 0) * 32 + lane, acc[i][k][0]);
          __stcg(slot + ((i * C::NI + k) * 2 + 1) * 32 + lane, acc[i][k][1]);
        }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release(&args.flags[cta * C::NCW + warp], 1);
      continue;
    }
    if (k0 > 0) {
      // owner: add the partials of the earlier CTAs in fixed order c-1, c-2, ...
      const int64_t it0 = base;
      int64_t cf = (it0 * args.G) / args.total;
      while (cf + 1 < args.G && range_start(cf + 1, args) <= it0) ++cf;
      while (cf > 0 && range_start(cf, args) > it0) --cf;
      for (int64_t c2 = int64_t(cta) - 1; c2 >= cf; --c2) {
        int* flag = &args.flags[c2 * C::NCW + warp];
        while (ld_acquire(flag) == 0) {
        }
        const double* slot = args.ws + (c2 * C::NCW + warp) * (C::FRAG * 32);
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int k = 0; k < C::NI; ++k) {
            acc[i][k][0] += __ldcg(slot + ((i * C::NI + k) * 2 + 0) * 32 + lane);
            acc[i][k][1] += __ldcg(slot + ((i * C::NI + k) * 2 + 1) * 32 + lane);
          }
        __syncwarp();
        if (lane == 0) *flag = 0;  // consumed; zero again for the next launch
      }
    }
    // store: lane (g, t) owns complex C[row g][col t] of each 8 x (4 complex) tile
    const int64_t b = tile / tiles_mn;
    const int64_t r = tile - b * tiles_mn;
    const int tn = int(r / args.tiles_m), tm = int(r - int64_t(tn) * args.tiles_m);
    double2* out = args.C + b * args.sCb;
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int64_t row = int64_t(tm) * C::BM + wm * C::WM + i * 8 + g;
      if (row >= args.M) continue;
#pragma unroll
      for (int k = 0; k < C::NI; ++k) {
        const int64_t col = int64_t(tn) * C::BN + wn * C::WN + k * 4 + t;
        if (col < args.Nn) out[row * args.ldc + col] = make_double2(acc[i][k][0], acc[i][k][1]);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map_box(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                  const uint32_t box_in[4]) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t gd[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t gs[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  cuuint32_t box[4] = {box_in[0], box_in[1], box_in[2], box_in[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), gd, gs, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
              uint32_t box1) {
  const uint32_t box[4] = {16, box1, 1, 1};
  return make_map_box(map, base, dims, strides_bytes, box);
}


template <class C>
void geometry(const ZgemmProblem& p, int num_sms, int& tiles_m, int& tiles_n, int& kt_per_o, int64_t& total,
              int& G) {
  tiles_m = int((p.M + C::BM - 1) / C::BM);
  tiles_n = int((p.Nn + C::BN - 1) / C::BN);
  kt_per_o = int((p.Kin + C::BK - 1) / C::BK);
  const int64_t KT = p.Ko * kt_per_o;
  total = int64_t(tiles_m) * tiles_n * p.batch * KT;
  G = int(total < num_sms ? total : num_sms);
}

// The flag region has a fixed size (max grid) so that it stays zero across problems that
// share a workspace: every launch leaves all its flags at zero.
template <class C>
size_t flag_bytes(int num_sms) {
  return ((size_t(num_sms) * C::NCW * 4 + 255) / 256) * 256;
}

template <class C>
size_t ws_bytes(const ZgemmProblem& p, int num_sms) {
  int tm, tn, kpo, G;
  int64_t total;
  geometry<C>(p, num_sms, tm, tn, kpo, total, G);
  const size_t slots = size_t(G) * C::SLOT_DOUBLES * 8;
  return flag_bytes<C>(num_sms) + slots;
}

template <class C>
cudaError_t launch_cfg(const ZgemmProblem& p, void* ws, size_t ws_size, int num_sms, cudaStream_t st, int* nl) {
  CUtensorMap ta, tb;
  const uint64_t sAo = p.Ko > 1 ? p.sAo : p.lda * p.M;
  const uint64_t sBo = p.Ko > 1 ? p.sBo : p.ldb * p.Kin;
  const uint64_t da[4] = {uint64_t(2 * p.Kin), uint64_t(p.M), uint64_t(p.Ko), uint64_t(p.batch)};
  const uint64_t sa[3] = {uint64_t(p.lda) * 16, sAo * 16, uint64_t(p.batch > 1 ? p.sAb : sAo * p.Ko) * 16};
  const uint64_t db[4] = {uint64_t(2 * p.Nn), uint64_t(p.Kin), uint64_t(p.Ko), uint64_t(p.batch)};
  const uint64_t sb[3] = {uint64_t(p.ldb) * 16, sBo * 16, uint64_t(p.batch > 1 ? p.sBb : sBo * p.Ko) * 16};
  if (!make_map(&ta, p.A, da, sa, C::BM) || !make_map(&tb, p.B, db, sb, C::BK)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(zgemm_dmma_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (ws == nullptr || ws_size < ws_bytes<C>(p, num_sms)) return cudaErrorInvalidValue;
  KArgs a;
  int G;
  geometry<C>(p, num_sms, a.tiles_m, a.tiles_n, a.kt_per_o, a.total, G);
  a.G = G;
  a.KT = int(p.Ko * a.kt_per_o);
  a.C = static_cast<double2*>(p.C);
  const size_t flags = flag_bytes<C>(num_sms);
  a.flags = static_cast<int*>(ws);
  a.ws = reinterpret_cast<double*>(static_cast<char*>(ws) + flags);
  a.M = p.M;
  a.Nn = p.Nn;
  a.ldc = p.ldc;
  a.sCb = p.sCb;
  zgemm_dmma_kernel<C><<<G, C::THREADS, C::SMEM, st>>>(ta, tb, a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && nl) ++*nl;
  return e;
}

}  // namespace

bool encode_map_4d(void* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                   const uint32_t box[4]) {
  return make_map_box(static_cast<CUtensorMap*>(map), base, dims, strides_bytes, box);
}

bool encode_zgemm_maps(void* mapA, void* mapB, const ZgemmProblem& p, int BM, int BK) {
  const uint64_t sAo = p.Ko > 1 ? p.sAo : p.lda * p.M;
  const uint64_t sBo = p.Ko > 1 ? p.sBo : p.ldb * p.Kin;
  const uint64_t da[4] = {uint64_t(2 * p.Kin), uint64_t(p.M), uint64_t(p.Ko), uint64_t(p.batch)};
  const uint64_t sa[3] = {uint64_t(p.lda) * 16, sAo * 16, uint64_t(p.batch > 1 ? p.sAb : sAo * p.Ko) * 16};
  const uint64_t db[4] = {uint64_t(2 * p.Nn), uint64_t(p.Kin), uint64_t(p.Ko), uint64_t(p.batch)};
  const uint64_t sb[3] = {uint64_t(p.ldb) * 16, sBo * 16, uint64_t(p.batch > 1 ? p.sBb : sBo * p.Ko) * 16};
  return make_map(static_cast<CUtensorMap*>(mapA), p.A, da, sa, uint32_t(BM)) &&
         make_map(static_cast<CUtensorMap*>(mapB), p.B, db, sb, uint32_t(BK));
}

cudaError_t zgemm_preload() {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, zgemm_dmma_kernel<Big>);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(zgemm_dmma_kernel<Big>, cudaFuncAttributeMaxDynamicSharedMemorySize, Big::SMEM);
}

size_t zgemm_workspace_bytes(const ZgemmProblem& p, int num_sms) { return ws_bytes<Big>(p, num_sms); }

cudaError_t launch_zgemm(const ZgemmProblem& p, void* workspace, size_t ws_size, int num_sms, cudaStream_t stream,
                         int* n_launches) {
  if (p.M <= 0 || p.Nn <= 0 || p.Kin <= 0 || p.Ko <= 0 || p.batch <= 0) return cudaErrorInvalidValue;
  if (2 * p.Kin > (int64_t(1) << 31) || p.M > (int64_t(1) << 31) || p.batch > (int64_t(1) << 31))
    return cudaErrorInvalidValue;
  return launch_cfg<Big>(p, workspace, ws_size, num_sms, stream, n_launches);
}

}  // namespace cc
