// Latency of the exact (fp64, reference-order) evaluator exact_u_fast on the
// device: one thread, then N entries spread over the grid (the fix-list
// pattern of k_spec_fix).  Build and run on the GPU box:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude \
//        -Ipaper_1409_7474_b200/csrc tools/exact_latency.cu -o /tmp/exact_latency && /tmp/exact_latency
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

#include "lse_b200.h"
#include "lse_device.cuh"
#include "lse_fast.cuh"

using namespace lse;

__global__ void k_eval(const ExactCtx* c, const uint32_t* bits, const int2* pts, int n, double* out,
                       int spread) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = spread ? threadIdx.x * gridDim.x + blockIdx.x : t;
  if (q >= n) return;
  out[q] = exact_u_fast<4, SRC_SMOOTH>(c, bits, pts[q].y, pts[q].x, false);
}

int main() {
  const int H = 4096, W = 4096, HR = H / 32, pitch = W;
  std::vector<uint32_t> bits((size_t)HR * pitch);
  unsigned s = 12345;
  for (auto& b : bits) { s = s * 1664525u + 1013904223u; b = s; }
  std::vector<float> img((size_t)H * W);
  for (auto& v : img) { s = s * 1664525u + 1013904223u; v = (s >> 8) * (1.0f / 16777216.0f); }
  uint32_t* dbits; float* dimg; ExactCtx* dctx; Scalars* dsc; double* dlut; double* dout; int2* dpts;
  cudaMalloc(&dbits, bits.size() * 4);
  cudaMalloc(&dimg, img.size() * 4);
  cudaMalloc(&dctx, sizeof(ExactCtx));
  cudaMalloc(&dsc, sizeof(Scalars));
  cudaMalloc(&dlut, 512 * 8);
  cudaMalloc(&dout, 65536 * 8);
  cudaMalloc(&dpts, 65536 * sizeof(int2));
  cudaMemcpy(dbits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dimg, img.data(), img.size() * 4, cudaMemcpyHostToDevice);
  std::vector<double> lut(512, 0.1);
  cudaMemcpy(dlut, lut.data(), 512 * 8, cudaMemcpyHostToDevice);
  Scalars sc;
  std::memset(&sc, 0, sizeof(sc));
  sc.c_pos = 0.7; sc.c_neg = 0.3; sc.dc = 0.4; sc.peak = 0.3; sc.model = REGION;
  cudaMemcpy(dsc, &sc, sizeof(sc), cudaMemcpyHostToDevice);
  ExactCtx c;
  std::memset(&c, 0, sizeof(c));
  c.H = H; c.W = W; c.R = 4; c.pitch_w = pitch; c.data_pitch = W; c.data32 = dimg;
  for (int d = 0; d <= 4; ++d) c.w64[d] = 0.2 / (1 + d);
  c.dt = 15.0; c.scal = dsc; c.model = REGION; c.lut64 = dlut;
  cudaMemcpy(dctx, &c, sizeof(c), cudaMemcpyHostToDevice);
  std::vector<int2> pts(65536);
  for (auto& p : pts) { s = s * 1664525u + 1013904223u; p.x = 8 + (s >> 8) % (W - 16); s = s * 1664525u + 1013904223u; p.y = 8 + (s >> 8) % (H - 16); }
  cudaMemcpy(dpts, pts.data(), pts.size() * sizeof(int2), cudaMemcpyHostToDevice);
  // the last 32 entries: border pixels (the general path)
  std::vector<int2> bpts(32);
  for (int k = 0; k < 32; ++k) bpts[k] = make_int2(100 + 7 * k, k % 3);
  cudaMemcpy(dpts + 65536 - 32, bpts.data(), 32 * sizeof(int2), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { int n, grid, block, spread; const char* name; } cases[] = {
      {1, 1, 32, 0, "1 entry"}, {32, 1, 32, 0, "32 entries, 1 warp"},
      {3000, 148, 256, 0, "3000 entries, blocks of 256 in order"},
      {3000, 148, 256, 1, "3000 entries spread over the grid"},
      {30000, 148, 256, 1, "30000 entries spread"}};
  struct Border { } ;
  for (auto& k : cases) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_eval<<<k.grid, k.block>>>(dctx, dbits, dpts, k.n, dout, k.spread);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) std::printf("%-40s %8.2f us\n", k.name, ms * 1e3);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_eval<<<1, 32>>>(dctx, dbits, dpts + 65536 - 32, 32, dout, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) std::printf("%-40s %8.2f us\n", "32 border entries (general path)", ms * 1e3);
  }
  std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
