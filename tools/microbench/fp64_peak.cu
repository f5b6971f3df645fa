// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Evidence for the FP64 roofline denominator used by bench.py / DESIGN.md.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;  // practically never; keeps the work alive
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters, double seed) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * 1e-3 + threadIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed - i * 1e-3;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
double run(K kern, int blocks, int threads, int iters, double flop_per_thread_iter, const char* name) {
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<blocks, threads>>>(out, iters / 10, 1.0);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(out, iters, 1.0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  double flops = flop_per_thread_iter * (double)blocks * threads * iters;
  double tf = flops / (best * 1e-3) / 1e12;
  printf("%-28s blocks=%5d threads=%4d  %.3f ms  %.2f TFLOP/s\n", name, blocks, threads, best, tf);
  CK(cudaFree(out));
  return tf;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, clk_khz);
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  // m8n8k4: 8*8*4 FMA per warp = 512 flop per warp per mma = 16 flop per thread per mma
  for (int w : {1, 2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "dmma m8n8k4 x8acc w=%d", w);
    run(dmma_m8n8k4<8>, sms, 32 * w, iters, 8 * 16.0, nm);
  }
  run(dmma_m8n8k4<4>, sms, 32 * 8, iters, 4 * 16.0, "dmma m8n8k4 x4acc w=8");
  run(dmma_m8n8k4<16>, sms, 32 * 8, iters, 16 * 16.0, "dmma m8n8k4 x16acc w=8");
  run(dmma_m8n8k4<8>, sms * 2, 32 * 8, iters, 8 * 16.0, "dmma m8n8k4 x8acc 2cta w=8");
  // m16n8k16: 16*8*16 FMA = 4096 flop per warp per mma = 128 flop per thread
  for (int w : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "dmma m16n8k16 x4acc w=%d", w);
    run(dmma_m16n8k16<4>, sms, 32 * w, iters / 4, 4 * 128.0, nm);
  }
  for (int w : {4, 8, 16, 32}) {
    char nm[64];
    snprintf(nm, 64, "dfma x8 w=%d", w);
    run(dfma_loop<8>, sms, 32 * w, iters * 4, 8 * 2.0, nm);
  }
  run(dfma_loop<8>, sms * 4, 256, iters * 4, 8 * 2.0, "dfma x8 4cta w=8");
  return 0;
}
