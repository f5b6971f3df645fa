// L2-hit read bandwidth: every CTA streams a slice of an L2-resident buffer (16-byte loads,
// __ldcg), many passes; and the same from a buffer larger than L2 (HBM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu && ./l2_bw
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ p, size_t n, int passes, double* out) {
  double s = 0;
  for (int k = 0; k < passes; ++k)
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
      double2 v = __ldcg(p + i);
      s += v.x + v.y;
    }
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  for (size_t mb : {16, 32, 64, 96, 4096}) {
    size_t n = (mb << 20) / 16;
    double2* p;
    cudaMalloc(&p, n * 16);
    cudaMemset(p, 0, n * 16);
    int passes = mb >= 1024 ? 2 : int(8192 / mb);
    for (int thr : {256, 512, 1024}) {
      for (int cps : {1, 2}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        rd<<<148 * cps, thr>>>(p, n, 1, out);
        cudaEventRecord(a);
        rd<<<148 * cps, thr>>>(p, n, passes, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("buffer %5zu MB threads %4d x %d CTA/SM: %.2f TB/s\n", mb, thr, cps, double(n * 16) * passes / (ms * 1e-3) / 1e12);
      }
    }
    cudaFree(p);
  }
  return 0;
}
