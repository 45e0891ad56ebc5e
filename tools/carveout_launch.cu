// Back-to-back launches of kernels with different shared-memory footprints:
// does switching the L1/shared carveout between kernels cost time?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 4) big(int* out, int n) {
  __shared__ float s[9728];                       // 38 KB
  s[threadIdx.x] = n;
  __syncthreads();
  if (n >= 0) out[0] = (int)s[(threadIdx.x + 1) % 128];
}
__global__ void small(int* out, int n) {
  if (n >= 0) out[0] = n;
}
int main() {
  int* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 2) {
      cudaFuncSetAttribute(small, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    for (int i = 0; i < 10; ++i) { big<<<40, 128>>>(d, -1); small<<<1, 1024>>>(d, -1); }
    cudaEventRecord(a);
    for (int i = 0; i < 200; ++i) {
      big<<<40, 128>>>(d, -1);
      if (mode >= 1) small<<<1, 1024>>>(d, -1);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (%s): %.2f us per iteration\n", mode,
           mode == 0 ? "big only" : mode == 1 ? "big+small default carveout" : "big+small carveout 100",
           ms * 1e3 / 200);
  }
  return 0;
}
