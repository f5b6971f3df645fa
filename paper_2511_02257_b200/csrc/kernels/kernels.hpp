// Device kernels of the contraction engine (sm_100a).  Host-callable launchers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cc {

// Batched complex (interleaved complex128) GEMM with a two-level K index:
//   C[b][m][n] = sum_{ko < Ko} sum_{ki < Kin} A[b][m][ko,ki] * B[b][ko,ki][n]
//   A(b,m,ko,ki) at A + b*sAb + ko*sAo + m*lda + ki      (complex-element strides)
//   B(b,ko,ki,n) at B + b*sBb + ko*sBo + ki*ldb + n
//   C(b,m,n)     at C + b*sCb + m*ldc + n
// MM1, BM1 and BB2 are all instances.  Runs on FP64 DMMA fed by TMA.
struct ZgemmProblem {
  const void* A;
  const void* B;
  void* C;
  int64_t M, Nn, Kin, Ko, batch;
  int64_t lda, sAo, sAb;
  int64_t ldb, sBo, sBb;
  int64_t ldc, sCb;
};

// TMA maps (CUtensorMap, 128 B each) of a problem's A and B for a BM x BK / BK x 8 box
// with 128-byte swizzle, as the DMMA kernels read them.
bool encode_zgemm_maps(void* mapA, void* mapB, const ZgemmProblem& p, int BM, int BK);

// A 4-d FP64 tensor map (dims[0] innermost, strides in bytes of dims 1..3, box extents),
// 128-byte swizzle.
bool encode_map_4d(void* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                   const uint32_t box[4]);

// Workspace bytes a problem needs for its deterministic split-K partials.
size_t zgemm_workspace_bytes(const ZgemmProblem& p, int num_sms);
cudaError_t launch_zgemm(const ZgemmProblem& p, void* workspace, size_t ws_bytes, int num_sms,
                         cudaStream_t stream, int* n_launches);

// "Contract all" of two nodes as a sum of traces of G strided N x N sub-matrices per time
// slice: c[t] = sum_g sum_{i,k} A[t](g)[i][k] B[t](g)[k][i] with X[t](g)[r][c] at
// X + t sT + (g / Gj) sGo + (g % Gj) sGi + r ld + c (complex elements).
//   TR_MM: G = 1, ld = N, sT = N^2.   BB3 (reading T4-3): g = (s, j), G = S N, Gj = N,
//   sGo = N^3, sGi = N, ld = N^2, sT = S N^3 (A_sj[i][k] = A[t,s,i,j,k], B_sj[k][i] = B[t,s,k,j,i]).
struct TraceShape {
  int64_t N, ld, sT, sGo, sGi;
  int32_t G, Gj;
};
TraceShape trace_shape(int op, int64_t N, int64_t S);   // op = CC_TR_MM or CC_BB3
// out[t] (complex128) written with a fixed-order reduction.  Workspace: counters (zero on entry,
// zero again on exit) + unit partials.
size_t trace_workspace_bytes(int64_t Lt, const TraceShape& sh);
cudaError_t launch_trace(const void* A, const void* B, void* out, int64_t Lt, const TraceShape& sh, void* workspace,
                         cudaStream_t stream);
// n <= trace_batch_max() traces of the same shape in one launch (out[k] = Lt complex128 each).
int trace_batch_max();
cudaError_t launch_trace_batch(const void* const* A, const void* const* B, void* const* out, int n, int64_t Lt,
                               const TraceShape& sh, void* workspace, cudaStream_t stream);

// corr[c][t] = sum over the terms of correlator c (in input order) of coef * roots[tree][t].
// term_start: n_corr+1 offsets into (term_tree, term_coef).
cudaError_t launch_correlate(const void* roots, void* corr, int64_t n_corr, int64_t Lt, const int32_t* term_start,
                             const int32_t* term_tree, const double* term_coef, cudaStream_t stream);

// Force-load the kernels of each translation unit (CUDA lazy loading would otherwise load a
// kernel at its first launch, which can wait for an idle device — a deadlock while copy
// streams wait on a persistent worker).  Also sets their shared-memory attributes.
// Copy bytes (multiple of 16, 16-byte aligned) from pinned host memory to device memory
// with SM loads over PCIe, ordered on `stream` (not behind pending copy-engine transfers).
cudaError_t launch_upload(void* dst, const void* src_pinned, size_t bytes, int num_sms, cudaStream_t stream);
cudaError_t zgemm_preload();
cudaError_t trace_preload();

// MM1 by Ozaki splitting on tcgen05 INT8 tensor cores (ozaki.cu): C[t] = A[t] B[t], complex128
// [Lt][N][N], n_slices in 4..8 INT8 slices per operand; workspace holds the slices + scales.
size_t ozaki_mm1_workspace_bytes(int64_t Lt, int64_t N, int slices);
// A pre-split operand: INT8 slices (tile-contiguous) + power-of-two exponents, in the A-form
// (rows of A_cat) or the B-form (columns of B_cat); made once and shared by every MM1 that
// reads the same tensor in the same role.
struct OzakiForm {
  const void* slices;
  const int* exps;
};
// Any MM1 / BM1 / BB2-shaped problem (ZgemmProblem layout, two-level K, batch = time
// slices): workspace for batches of up to max_batch slices; forms of the full batch.
size_t ozaki_workspace_bytes(const ZgemmProblem& q, int slices, int64_t max_batch);
size_t ozaki_form_bytes(const ZgemmProblem& q, int slices, bool as_b);
cudaError_t launch_ozaki_form(const ZgemmProblem& q, int slices, bool as_b, void* dst, OzakiForm* form,
                              cudaStream_t stream);
cudaError_t launch_ozaki_gemm(const ZgemmProblem& q, int slices, void* ws, size_t ws_bytes, cudaStream_t stream,
                              const OzakiForm* fa = nullptr, const OzakiForm* fb = nullptr);
// fa / fb: pre-split operands (nullptr: split A / B into the workspace first).
cudaError_t launch_ozaki_mm1(const void* A, const void* B, void* C, int64_t Lt, int64_t N, int slices, void* ws,
                             size_t ws_bytes, cudaStream_t stream, const OzakiForm* fa = nullptr,
                             const OzakiForm* fb = nullptr);
// Plain INT8 GEMM on the same tcgen05 machinery: C[m][n] = sum_k A[m][k] B[n][k] (int32).
cudaError_t launch_i8gemm_tn(const int8_t* A, const int8_t* B, int32_t* C, int64_t M, int64_t Nn, int64_t K,
                             cudaStream_t stream);

// Synthetic leaf values (input generation; same recipe as synth/rng.py).
cudaError_t launch_fill_synthetic(void* dev, int64_t n, uint64_t seed, int64_t leaf_id, int64_t e0, int mode,
                                  double sigma, cudaStream_t stream);

}  // namespace cc
