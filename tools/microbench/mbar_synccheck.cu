// Does compute-sanitizer synccheck report "Missing init" for mbarrier.test_wait on a static
// shared-memory mbarrier initialised by thread 0 before __syncthreads (the dataflow worker's
// done[] / info_full[] pattern)?  Variant v: 0 = as in dataflow.cu (init loop + fence +
// test_wait poll), 1 = no fence.mbarrier_init, 2 = try_wait instead of test_wait.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__global__ void k(int v, int* out) {
  __shared__ uint64_t bars[2][4];
  __shared__ double red[4][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int x = 0; x < 2; ++x)
      for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bars[x][s])), "r"(1));
    if (v != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < 4; ++s) {
      red[s][0] = s + 1.0;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bars[0][s])) : "memory");
    }
  }
  if (warp == 2 && lane == 0) {
    double sum = 0;
    for (int s = 0; s < 4; ++s) {
      uint32_t ok = 0;
      while (!ok) {
        if (v == 2)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                       : "=r"(ok) : "r"(sa(&bars[0][s])), "r"(0) : "memory");
        else
          asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                       : "=r"(ok) : "r"(sa(&bars[0][s])), "r"(0) : "memory");
      }
      sum += red[s][0];
    }
    out[blockIdx.x] = int(sum);
  }
}
int main(int argc, char** argv) {
  int v = argc > 1 ? atoi(argv[1]) : 0;
  int* d;
  cudaMalloc(&d, 4 * 148);
  k<<<148, 128>>>(v, d);
  cudaError_t e = cudaDeviceSynchronize();
  int h = 0;
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("variant %d: %s, out %d (want 10)\n", v, cudaGetErrorString(e), h);
  return 0;
}
