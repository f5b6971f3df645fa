// "Contract all" for tree roots and the correlator sums.
//
// TR_MM: c[t] = sum_{i,j} A[t,i,j] * B[t,j,i]  (reading V-1).  HBM/L2-bound (0.25 flop/B).
// BB3 (reading T4-3): c[t] = sum_s sum_{i,j,k} A[t,s,i,j,k] B[t,s,k,j,i] is the same operation
// over G = S N strided sub-matrices per slice: for each (s, j), A_sj[i][k] = A[t,s,i,j,k] and
// B_sj[k][i] = B[t,s,k,j,i] are N x N matrices with row stride N^2, and c[t] = sum over (s, j)
// of tr(A_sj B_sj) (TraceShape, kernels.hpp).
// Work unit = (t, g, I, J): the 32x32 complex block A[t, I, J] of sub-matrix g and its transpose partner
// B[t, J, I] (16 KB each, coalesced 512-byte row segments).  Slice t is split into P
// pieces of consecutive units (P chosen so Lt*P ~ 2 CTAs per SM); CTA (t, p) walks its
// units with the next unit's eight 16-byte loads per thread issued before the current
// unit is consumed (software prefetch keeps ~8 KB per warp in flight), transposes B's block
// through padded shared memory (conflict-free) and accumulates per thread.  The CTA partial
// is reduced in a fixed order (shuffle tree, then warps in order) into partials[t][p]; the
// last CTA of slice t (ticket counter) sums the P partials in order.  No floating-point
// atomics: the result is bit-identical from run to run.
#include <algorithm>

#include "cc.h"
#include "kernels.hpp"

namespace cc {
namespace {

#ifndef TR_MINB
#define TR_MINB 2
#endif
constexpr int TB = 32;          // block edge (complex elements)
constexpr int TRB = 32;         // traces per batched launch
constexpr int TR_THREADS = 256; // 8 warps; warp w owns rows w, w+8, w+16, w+24 of a block
constexpr int RPW = TB / 8;     // rows per warp

__device__ __forceinline__ double2 cmul_acc(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}

__device__ __forceinline__ void load_unit(const double2* __restrict__ At, const double2* __restrict__ Bt,
                                          const TraceShape& sh, int nb, int unit, int warp, int lane,
                                          double2 (&a)[RPW], double2 (&b)[RPW]) {
  const int nb2 = nb * nb;
  const int g = unit / nb2, rem = unit - g * nb2;
  const int I = rem / nb, J = rem - I * nb;
  const int64_t N = sh.N, ld = sh.ld;
  const int64_t goff = int64_t(g / sh.Gj) * sh.sGo + int64_t(g % sh.Gj) * sh.sGi;   // sub-matrix g
  const int64_t i0 = int64_t(I) * TB, j0 = int64_t(J) * TB;
#pragma unroll
  for (int rr = 0; rr < RPW; ++rr) {
    const int r = warp + rr * 8;
    const int64_t ia = i0 + r, ja = j0 + lane;   // A_g[I0 + r, J0 + lane]
    const int64_t jb = j0 + r, ib = i0 + lane;   // B_g[J0 + r, I0 + lane]
    a[rr] = (ia < N && ja < N) ? __ldg(At + goff + ia * ld + ja) : make_double2(0.0, 0.0);
    b[rr] = (jb < N && ib < N) ? __ldg(Bt + goff + jb * ld + ib) : make_double2(0.0, 0.0);
  }
}

// Up to TRB traces per launch (blockIdx.z): consecutive TR_MM ops of a plan share one launch,
// so the ramp-up and tail of a launch are paid once per batch.
struct TraceBatch {
  const double2* A[TRB];
  const double2* B[TRB];
  double2* out[TRB];
};

__global__ void __launch_bounds__(TR_THREADS, TR_MINB)
    trace_kernel(const __grid_constant__ TraceBatch tb, const TraceShape sh, int nb, int P,
                 double2* __restrict__ partials, int* __restrict__ counters) {
  __shared__ double2 sB[TB][TB + 1];
  __shared__ double2 red[TR_THREADS / 32];
  __shared__ int is_last;
  const int t = blockIdx.y, p = blockIdx.x, z = blockIdx.z;
  const double2* __restrict__ A = tb.A[z];
  const double2* __restrict__ B = tb.B[z];
  double2* __restrict__ out = tb.out[z];
  partials += int64_t(z) * gridDim.y * P;
  counters += int64_t(z) * gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int U = sh.G * nb * nb;
  const int u0 = int((int64_t(p) * U) / P), u1 = int((int64_t(p + 1) * U) / P);
  const double2* At = A + int64_t(t) * sh.sT;
  const double2* Bt = B + int64_t(t) * sh.sT;
  double2 acc = make_double2(0.0, 0.0);
  double2 a[RPW], b[RPW], an[RPW], bn[RPW];
  if (u0 < u1) load_unit(At, Bt, sh, nb, u0, warp, lane, a, b);
  for (int u = u0; u < u1; ++u) {
    if (u + 1 < u1) load_unit(At, Bt, sh, nb, u + 1, warp, lane, an, bn);
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) sB[warp + rr * 8][lane] = b[rr];
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) acc = cmul_acc(acc, a[rr], sB[lane][warp + rr * 8]);  // B[J0+lane][I0+r]
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
      a[rr] = an[rr];
      b[rr] = bn[rr];
    }
  }
  // fixed-order CTA reduction
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = red[0];
    for (int w = 1; w < TR_THREADS / 32; ++w) {
      s.x += red[w].x;
      s.y += red[w].y;
    }
    if (P == 1) {
      out[t] = s;
      is_last = 0;
    } else {
      partials[int64_t(t) * P + p] = s;
      __threadfence();
      const int ticket = atomicAdd(&counters[t], 1);
      is_last = (ticket == P - 1);
    }
  }
  __syncthreads();
  if (is_last) {
    // last CTA of slice t: fixed-order sum of the P partials (lane-strided partial sums,
    // then a shuffle tree; the order depends only on P)
    __threadfence();
    if (warp == 0) {
      const volatile double* pp = reinterpret_cast<const volatile double*>(partials + int64_t(t) * P);
      double sx = 0.0, sy = 0.0;
      for (int k = lane; k < P; k += 32) {
        sx += pp[2 * k];
        sy += pp[2 * k + 1];
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if (lane == 0) {
        out[t] = make_double2(sx, sy);
        counters[t] = 0;  // ready for the next launch
      }
    }
  }
}

// Pieces per time slice: from P0 = slots / slices (one wave) upwards, the smallest P whose CTAs
// fill whole waves to within 5 % while each CTA keeps >= 16 units (else the least wasteful);
// e.g. 512 slices in 512 CTAs is a 1.7-wave launch that idles a third of its last wave.
int trace_pieces(int64_t Lt, const TraceShape& sh, int n_traces = 1) {
  const int64_t nb = (sh.N + TB - 1) / TB, U = int64_t(sh.G) * nb * nb;
  const int64_t slots = int64_t(TR_MINB) * 148, X = Lt * n_traces;
  const int64_t P0 = std::max<int64_t>(1, slots / X);
  int64_t P = P0;
  double best_waste = 1e9;
  for (int64_t q = P0; q <= P0 + 64 && (q == P0 || q * 16 <= U); ++q) {
    const int64_t ctas = X * q;
    const double waste = double((ctas + slots - 1) / slots * slots) / double(ctas) - 1.0;
    if (waste < best_waste - 1e-12) {
      P = q;
      best_waste = waste;
    }
    if (waste < 0.05) break;
  }
  if (P > U) P = U;
  if (P < 1) P = 1;
  return int(P);
}

// corr[c][t] = sum over terms of c (input order) of coef * roots[tree][t].  One CTA per
// correlator; its term list is staged through shared memory in chunks and the threads run
// over t, so root loads are coalesced across t.
constexpr int CORR_CHUNK = 256;

__global__ void correlate_kernel(const double2* __restrict__ roots, double2* __restrict__ corr, int64_t n_corr,
                                 int64_t Lt, const int32_t* __restrict__ term_start,
                                 const int32_t* __restrict__ term_tree, const double* __restrict__ term_coef) {
  __shared__ int32_t s_tree[CORR_CHUNK];
  __shared__ double2 s_coef[CORR_CHUNK];
  const int64_t c = blockIdx.x;
  const int k0 = term_start[c], k1 = term_start[c + 1];
  for (int64_t tb = 0; tb < Lt; tb += blockDim.x) {
    const int64_t t = tb + threadIdx.x;
    double re = 0.0, im = 0.0;
    for (int kc = k0; kc < k1; kc += CORR_CHUNK) {
      const int n = (k1 - kc) < CORR_CHUNK ? (k1 - kc) : CORR_CHUNK;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s_tree[i] = term_tree[kc + i];
        s_coef[i] = make_double2(term_coef[2 * (kc + i)], term_coef[2 * (kc + i) + 1]);
      }
      __syncthreads();
      if (t < Lt) {
        for (int i = 0; i < n; ++i) {
          const double2 r = roots[int64_t(s_tree[i]) * Lt + t];
          const double2 cf = s_coef[i];
          re += cf.x * r.x - cf.y * r.y;
          im += cf.x * r.y + cf.y * r.x;
        }
      }
    }
    if (t < Lt) corr[c * Lt + t] = make_double2(re, im);
  }
}

// ---- synthetic inputs (input generation only; recipe of synth/rng.py) ------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void fill_synthetic_kernel(double2* out, int64_t n, uint64_t key, int64_t e0, int mode, double sigma) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = 2 * uint64_t(e0 + i);
    const double u1 = __dmul_rn(double(splitmix64(key + j) >> 11), 0x1.0p-53);
    const double u2 = __dmul_rn(double(splitmix64(key + j + 1) >> 11), 0x1.0p-53);
    double re, im;
    if (mode == 0) {
      re = __dmul_rn(__dadd_rn(0.75, __dmul_rn(0.5, u1)), sigma);
      im = __dmul_rn(__dmul_rn(__dadd_rn(__dmul_rn(0.5, u2), -0.25), 0.5), sigma);
    } else {
      re = __dmul_rn(__dadd_rn(__dmul_rn(2.0, u1), -1.0), sigma);
      im = __dmul_rn(__dadd_rn(__dmul_rn(2.0, u2), -1.0), sigma);
    }
    out[i] = make_double2(re, im);
  }
}

}  // namespace

__global__ void upload_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16);

cudaError_t trace_preload() {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, trace_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, correlate_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, fill_synthetic_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, upload_kernel);
  return e;
}

// layout: counters (TRB x Lt ints, left at zero by every launch) then the unit partials (the
// most any batch of n <= TRB traces needs, n Lt P_n)
TraceShape trace_shape(int op, int64_t N, int64_t S) {
  if (op == CC_BB3) return TraceShape{N, N * N, S * N * N * N, N * N * N, N, int32_t(S * N), int32_t(N)};
  return TraceShape{N, N, N * N, 0, 0, 1, 1};
}

size_t trace_workspace_bytes(int64_t Lt, const TraceShape& sh) {
  size_t parts = 0;
  for (int n = 1; n <= TRB; ++n) parts = std::max(parts, size_t(n) * size_t(Lt * trace_pieces(Lt, sh, n)));
  return parts * 16 + ((size_t(TRB) * Lt * 4 + 255) / 256) * 256;
}

int trace_batch_max() { return TRB; }

cudaError_t launch_trace_batch(const void* const* A, const void* const* B, void* const* out, int n, int64_t Lt,
                               const TraceShape& sh, void* workspace, cudaStream_t stream) {
  if (Lt <= 0 || sh.N <= 0 || sh.G <= 0 || sh.Gj <= 0 || Lt > 65535 || n <= 0 || n > TRB) return cudaErrorInvalidValue;
  const int nb = int((sh.N + TB - 1) / TB);
  if (int64_t(sh.G) * nb * nb >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  const int P = trace_pieces(Lt, sh, n);
  int* counters = static_cast<int*>(workspace);
  double2* partials =
      reinterpret_cast<double2*>(static_cast<char*>(workspace) + ((size_t(TRB) * Lt * 4 + 255) / 256) * 256);
  TraceBatch tb{};
  for (int k = 0; k < n; ++k) {
    tb.A[k] = static_cast<const double2*>(A[k]);
    tb.B[k] = static_cast<const double2*>(B[k]);
    tb.out[k] = static_cast<double2*>(out[k]);
  }
  dim3 grid{unsigned(P), unsigned(Lt), unsigned(n)};
  trace_kernel<<<grid, TR_THREADS, 0, stream>>>(tb, sh, nb, P, partials, counters);
  return cudaGetLastError();
}

cudaError_t launch_trace(const void* A, const void* B, void* out, int64_t Lt, const TraceShape& sh, void* workspace,
                         cudaStream_t stream) {
  return launch_trace_batch(&A, &B, &out, 1, Lt, sh, workspace, stream);
}

cudaError_t launch_correlate(const void* roots, void* corr, int64_t n_corr, int64_t Lt, const int32_t* term_start,
                             const int32_t* term_tree, const double* term_coef, cudaStream_t stream) {
  if (n_corr <= 0 || Lt <= 0) return cudaSuccess;
  const int threads = Lt >= 256 ? 256 : int((Lt + 31) / 32 * 32);
  correlate_kernel<<<unsigned(n_corr), threads, 0, stream>>>(static_cast<const double2*>(roots), static_cast<double2*>(corr), n_corr,
                                               Lt, term_start, term_tree, term_coef);
  return cudaGetLastError();
}

// SM-driven upload from pinned host memory (UVA) to device memory: a stream-ordered copy
// that does not queue behind the copy engines' pending transfers (the leaf H2D copies).
__global__ void upload_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_upload(void* dst, const void* src_pinned, size_t bytes, int num_sms, cudaStream_t stream) {
  if (bytes == 0) return cudaSuccess;
  if ((bytes & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src_pinned) & 15))
    return cudaErrorInvalidValue;
  const int64_t n16 = int64_t(bytes / 16);
  const int64_t blocks = std::min<int64_t>(int64_t(num_sms) * 4, (n16 + 255) / 256);
  upload_kernel<<<unsigned(blocks), 256, 0, stream>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src_pinned), n16);
  return cudaGetLastError();
}

cudaError_t launch_fill_synthetic(void* dev, int64_t n, uint64_t seed, int64_t leaf_id, int64_t e0, int mode,
                                  double sigma, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const uint64_t hkey = splitmix64(splitmix64(seed) ^ uint64_t(leaf_id));
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_synthetic_kernel<<<unsigned(blocks), 256, 0, stream>>>(static_cast<double2*>(dev), n, hkey, e0, mode, sigma);
  return cudaGetLastError();
}

}  // namespace cc
