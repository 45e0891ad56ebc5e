// Launch cost vs per-thread local memory (stack) size, stack reserved but untouched.
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__global__ void __launch_bounds__(128, 4) k(int* out, int n) {
  if (n >= 0) {                        // never taken at run time
    volatile int buf[N];
    for (int i = 0; i < N; ++i) buf[i] = i * threadIdx.x + n;
    int s = 0;
    for (int i = 0; i < N; ++i) s += buf[(i * 7) % N];
    out[0] = s;
  }
}
template <int N>
void run(int grid) {
  int* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) k<N><<<grid, 128>>>(d, -1);
  cudaEventRecord(a);
  for (int i = 0; i < 200; ++i) k<N><<<grid, 128>>>(d, -1);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("stack %5d B grid %4d: %.2f us/launch\n", N * 4, grid, ms * 1e3 / 200);
  cudaFree(d);
}
int main() {
  for (int g : {40, 592}) { run<1>(g); run<64>(g); run<300>(g); run<1000>(g); }
  return 0;
}
