// Per-SM TMA ingest from L2: one producer thread per CTA (grid = 148) streams 32 KB stages
// through a ring of S stages (no consumer math), for several stage shapes:
//   0: 8 tensor boxes of 32 rows x 128 B (SWIZZLE_128B; the df_worker trace stage)
//   1: 2 tensor boxes of 128 rows x 128 B
//   2: one 1-D cp.async.bulk of 32 KB
//   3: 8 1-D cp.async.bulk of 4 KB
//   4: 1 box of 128 rows x 128 B + one 1-D bulk of 16 KB (column-panel trace stage)
//   5: 2 boxes of 64 rows x 128 B + 8 boxes of 16 rows x 128 B (the df_worker GEMM stage)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void box(void* d, const CUtensorMap* m, uint32_t b, int c, int r) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(sa(d)), "l"(m), "r"(b), "r"(c), "r"(r) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, int n, uint32_t b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sa(d)), "l"(s), "r"(n), "r"(b) : "memory");
}
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap m128,
                                          const __grid_constant__ CUtensorMap m64, const __grid_constant__ CUtensorMap m16,
                                          const char* buf, size_t bytes, int mode, int S, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x) return;
  char* st0 = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t nst = bytes / 32768;
  const int rows_total = int(bytes / 2048);
  auto issue = [&](int s, long long i) {
    const size_t g = (size_t(blockIdx.x) * 977 + size_t(i) * 148) % nst;
    uint32_t b = sa(&bar[s]);
    char* d = st0 + s * 32768;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], 32768;" ::"r"(b));
    const int r0 = int((g * 16) % (rows_total - 256));
    if (mode == 0) {
      for (int j = 0; j < 8; ++j) box(d + j * 4096, &m32, b, 16 * j, r0);
    } else if (mode == 1) {
      for (int j = 0; j < 2; ++j) box(d + j * 16384, &m128, b, 16 * j, r0);
    } else if (mode == 2) {
      bulk(d, buf + g * 32768, 32768, b);
    } else if (mode == 3) {
      for (int j = 0; j < 8; ++j) bulk(d + j * 4096, buf + g * 32768 + j * 4096, 4096, b);
    } else if (mode == 4) {
      box(d, &m128, b, 16 * int(g % 16), r0);
      bulk(d + 16384, buf + ((g + 7) % nst) * 32768, 16384, b);
    } else {
      for (int j = 0; j < 2; ++j) box(d + j * 8192, &m64, b, 16 * j, r0);
      for (int j = 0; j < 8; ++j) box(d + 16384 + j * 2048, &m16, b, 16 * j, r0 + 64);
    }
  };
  for (int s = 0; s < S; ++s) issue(s, s);
  unsigned long long acc = 0;
  for (long long i = 0; i < iters; ++i) {
    const int s = int(i % S);
    const uint32_t par = uint32_t((i / S) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(sa(&bar[s])), "r"(par) : "memory");
    acc += *reinterpret_cast<volatile unsigned long long*>(st0 + s * 32768);
    if (i + S < iters) issue(s, i + S);
  }
  if (acc == 1) sink[0] = acc;
}
static CUtensorMap mk(char* buf, size_t bytes, int rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {256, bytes / 2048};
  cuuint64_t str[1] = {2048};
  cuuint32_t bx[2] = {16, cuuint32_t(rows)};
  cuuint32_t es[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    printf("encode failed\n");
  return m;
}
int main() {
  const size_t bytes = 64ull << 20;
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  CUtensorMap m32 = mk(buf, bytes, 32), m128 = mk(buf, bytes, 128), m64 = mk(buf, bytes, 64), m16 = mk(buf, bytes, 16);
  const char* names[] = {"8 boxes 32r (trace stage now)", "2 boxes 128r", "bulk 32 KB", "8 bulk 4 KB",
                         "box 128r + bulk 16 KB (panel trace)", "2 boxes 64r + 8 boxes 16r (GEMM now)"};
  for (int mode = 0; mode < 6; ++mode)
    for (int S : {3, 6}) {
      const int smem = S * 32768 + 1024, iters = 4000;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k<<<148, 32, smem>>>(m32, m128, m64, m16, buf, bytes, mode, S, 100, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<148, 32, smem>>>(m32, m128, m64, m16, buf, bytes, mode, S, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      printf("%-40s S=%d %6.2f TB/s %5.1f B/cycle/SM %5.0f cycles/stage %s\n", names[mode], S,
             148.0 * iters * 32768 / (ms * 1e-3) / 1e12, 32768.0 * iters / (ms * 1e-3) / 1.965e9,
             (ms * 1e-3) * 1.965e9 / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
