// "Contract all" for tree roots and the correlator sums.
//
// TR_MM: c[t] = sum_{i,j} A[t,i,j] * B[t,j,i]  (reading V-1).  HBM/L2-bound (0.25 flop/B).
// Work unit = (t, I, J): the 32x32 complex block A[t, I, J] and its transpose partner
// B[t, J, I] (16 KB each, coalesced 512-byte row segments).  One CTA per unit, so every
// thread issues its 8 independent 16-byte loads up front and the whole GPU keeps
// megabytes in flight; B's block is transposed through padded shared memory
// (conflict-free).  The unit partial is reduced in a fixed order (warp shuffle tree, then
// warps in order) into partials[t][unit]; the last CTA of a time slice (ticket counter)
// sums the partials in unit order.  No floating-point atomics: the result is bit-identical
// from run to run.
#include "kernels.hpp"

namespace cc {
namespace {

constexpr int TB = 32;          // block edge (complex elements)
constexpr int TR_THREADS = 256; // 8 warps; warp w owns rows w, w+8, w+16, w+24 of a block

__device__ __forceinline__ double2 cmul_acc(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}

__global__ void __launch_bounds__(TR_THREADS)
    trace_kernel(const double2* __restrict__ A, const double2* __restrict__ B, double2* __restrict__ out, int64_t N,
                 int nb, double2* __restrict__ partials, int* __restrict__ counters) {
  __shared__ double2 sB[TB][TB + 1];
  __shared__ double2 red[TR_THREADS / 32];
  __shared__ int is_last;
  const int t = blockIdx.y;
  const int unit = blockIdx.x;            // unit = I * nb + J
  const int I = unit / nb, J = unit - I * nb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = int64_t(I) * TB, j0 = int64_t(J) * TB;
  const double2* At = A + int64_t(t) * N * N;
  const double2* Bt = B + int64_t(t) * N * N;
  double2 a[TB / 8], b[TB / 8];
#pragma unroll
  for (int rr = 0; rr < TB / 8; ++rr) {
    const int r = warp + rr * 8;
    const int64_t ia = i0 + r, ja = j0 + lane;   // A[t, I0 + r, J0 + lane]
    const int64_t jb = j0 + r, ib = i0 + lane;   // B[t, J0 + r, I0 + lane]
    a[rr] = (ia < N && ja < N) ? __ldg(At + ia * N + ja) : make_double2(0.0, 0.0);
    b[rr] = (jb < N && ib < N) ? __ldg(Bt + jb * N + ib) : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int rr = 0; rr < TB / 8; ++rr) sB[warp + rr * 8][lane] = b[rr];
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int rr = 0; rr < TB / 8; ++rr) acc = cmul_acc(acc, a[rr], sB[lane][warp + rr * 8]);  // B[J0+lane][I0+r]
  // fixed-order CTA reduction
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  const int nunits = nb * nb;
  if (threadIdx.x == 0) {
    double2 s = red[0];
    for (int w = 1; w < TR_THREADS / 32; ++w) {
      s.x += red[w].x;
      s.y += red[w].y;
    }
    if (nunits == 1) {
      out[t] = s;
      is_last = 0;
    } else {
      partials[int64_t(t) * nunits + unit] = s;
      __threadfence();
      const int ticket = atomicAdd(&counters[t], 1);
      is_last = (ticket == nunits - 1);
    }
  }
  __syncthreads();
  if (is_last) {
    // last CTA of slice t: fixed-order sum of the unit partials (warp 0: lane-strided
    // partial sums, then a shuffle tree; the order depends only on nunits)
    __threadfence();
    if (warp == 0) {
      const volatile double* pp = reinterpret_cast<const volatile double*>(partials + int64_t(t) * nunits);
      double sx = 0.0, sy = 0.0;
      for (int k = lane; k < nunits; k += 32) {
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

// corr[c][t] = sum over terms of c (input order) of coef * roots[tree][t]
__global__ void correlate_kernel(const double2* __restrict__ roots, double2* __restrict__ corr, int64_t n_corr,
                                 int64_t Lt, const int32_t* __restrict__ term_start,
                                 const int32_t* __restrict__ term_tree, const double* __restrict__ term_coef) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= n_corr * Lt) return;
  const int64_t c = e / Lt, t = e - c * Lt;
  double re = 0.0, im = 0.0;
  for (int k = term_start[c]; k < term_start[c + 1]; ++k) {
    const double2 r = roots[int64_t(term_tree[k]) * Lt + t];
    const double cr = term_coef[2 * k], ci = term_coef[2 * k + 1];
    // (cr + i ci)(r.x + i r.y), each term rounded as the oracle does: coef * root, then add
    const double pr = cr * r.x - ci * r.y;
    const double pi = cr * r.y + ci * r.x;
    re += pr;
    im += pi;
  }
  corr[e] = make_double2(re, im);
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

size_t trace_workspace_bytes(int64_t Lt, int64_t N) {
  const int64_t nb = (N + TB - 1) / TB;
  return size_t(Lt * nb * nb) * 16 + size_t(Lt) * sizeof(int) + 256;
}

cudaError_t launch_trace(const void* A, const void* B, void* out, int64_t Lt, int64_t N, void* workspace,
                         cudaStream_t stream) {
  if (Lt <= 0 || N <= 0 || Lt > 65535) return cudaErrorInvalidValue;
  const int nb = int((N + TB - 1) / TB);
  // layout: counters (Lt ints, left at zero by every launch) then the unit partials
  int* counters = static_cast<int*>(workspace);
  double2* partials = reinterpret_cast<double2*>(static_cast<char*>(workspace) + ((size_t(Lt) * 4 + 255) / 256) * 256);
  dim3 grid{unsigned(nb * nb), unsigned(Lt), 1u};
  trace_kernel<<<grid, TR_THREADS, 0, stream>>>(static_cast<const double2*>(A), static_cast<const double2*>(B),
                                               static_cast<double2*>(out), N, nb, partials, counters);
  return cudaGetLastError();
}

cudaError_t launch_correlate(const void* roots, void* corr, int64_t n_corr, int64_t Lt, const int32_t* term_start,
                             const int32_t* term_tree, const double* term_coef, cudaStream_t stream) {
  const int64_t total = n_corr * Lt;
  if (total <= 0) return cudaSuccess;
  const int blocks = int((total + 255) / 256);
  correlate_kernel<<<blocks, 256, 0, stream>>>(static_cast<const double2*>(roots), static_cast<double2*>(corr), n_corr,
                                               Lt, term_start, term_tree, term_coef);
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
