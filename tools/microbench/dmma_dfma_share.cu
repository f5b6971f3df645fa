// Does a DFMA stream starve when DMMA saturates the same SM?  One DMMA CTA (9 warps) and one
// DFMA CTA (4 warps) per SM, on two streams; DFMA throughput alone vs concurrent.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_dfma_share dmma_dfma_share.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(288, 1) dmma_kernel(double* out, int iters, int nap) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
    if (nap && (it & 63) == 0) __nanosleep(nap);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(128, 1) dfma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a0, a1, b0, b1;
  for (auto* ev : {&a0, &a1, &b0, &b1}) CK(cudaEventCreate(ev));
  const int sms = 148;
  const int it_dmma = 40000, it_dfma = 20000;
  dmma_kernel<<<sms, 288, 0, s1>>>(out, 100, 0);
  dfma_kernel<<<sms, 128, 0, s2>>>(out, 100);
  CK(cudaDeviceSynchronize());
  float ms;
  // alone
  CK(cudaEventRecord(b0, s2));
  dfma_kernel<<<sms, 128, 0, s2>>>(out, it_dfma);
  CK(cudaEventRecord(b1, s2));
  CK(cudaEventSynchronize(b1));
  CK(cudaEventElapsedTime(&ms, b0, b1));
  double dfma_flop = 2.0 * 8 * it_dfma * 128.0 * sms;
  printf("DFMA alone:      %.3f ms  %.2f TF/s\n", ms, dfma_flop / ms / 1e9);
  CK(cudaEventRecord(a0, s1));
  dmma_kernel<<<sms, 288, 0, s1>>>(out, it_dmma, 0);
  CK(cudaEventRecord(a1, s1));
  CK(cudaEventSynchronize(a1));
  CK(cudaEventElapsedTime(&ms, a0, a1));
  double dmma_flop = 512.0 * 8 * it_dmma * 9 * sms;
  printf("DMMA alone:      %.3f ms  %.2f TF/s\n", ms, dmma_flop / ms / 1e9);
  for (int nap : {0, 50, 200, 1000}) {
  printf("-- nap %d ns every 64 DMMA iterations\n", nap);
  CK(cudaEventRecord(a0, s1));
  dmma_kernel<<<sms, 288, 0, s1>>>(out, it_dmma, nap);
  CK(cudaEventRecord(a1, s1));
  CK(cudaEventRecord(b0, s2));
  dfma_kernel<<<sms, 128, 0, s2>>>(out, it_dfma);
  CK(cudaEventRecord(b1, s2));
  CK(cudaDeviceSynchronize());
  CK(cudaEventElapsedTime(&ms, b0, b1));
  printf("DFMA concurrent: %.3f ms  %.2f TF/s\n", ms, dfma_flop / ms / 1e9);
  CK(cudaEventElapsedTime(&ms, a0, a1));
  printf("DMMA concurrent: %.3f ms  %.2f TF/s\n", ms, dmma_flop / ms / 1e9);
  }
  // DFMA launched first
  CK(cudaEventRecord(b0, s2));
  dfma_kernel<<<sms, 128, 0, s2>>>(out, it_dfma * 20);
  CK(cudaEventRecord(b1, s2));
  CK(cudaEventRecord(a0, s1));
  dmma_kernel<<<sms, 288, 0, s1>>>(out, it_dmma, 0);
  CK(cudaEventRecord(a1, s1));
  CK(cudaDeviceSynchronize());
  CK(cudaEventElapsedTime(&ms, b0, b1));
  printf("DFMA-first: DFMA %.3f ms  %.2f TF/s", ms, 20 * dfma_flop / ms / 1e9);
  CK(cudaEventElapsedTime(&ms, a0, a1));
  printf("  DMMA %.3f ms  %.2f TF/s\n", ms, dmma_flop / ms / 1e9);
  return 0;
}
