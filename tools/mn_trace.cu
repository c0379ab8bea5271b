// mn_trace.cu -- timeline of one CTA of the MN-major (weight-gradient) kernel
// on the DNN A FC wgrad shape.  Debug tool, not product.
#define GA3C_TRACE 1
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "tc_ws.cuh"
using namespace ga3c;

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 40, IN = 2592, OUT = 256;
  std::vector<float> x((size_t)B * IN), d((size_t)B * OUT);
  for (size_t i = 0; i < x.size(); ++i) x[i] = (float)((i * 7919) % 1000) / 1000.f;
  for (size_t i = 0; i < d.size(); ++i) d[i] = (float)((i * 104729) % 1000) / 1000.f - 0.5f;
  float *dx, *dd, *dg; int* flag;
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&dd, d.size() * 4); cudaMalloc(&dg, (size_t)OUT * (IN + 1) * 4);
  cudaMalloc(&flag, 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, d.data(), d.size() * 4, cudaMemcpyHostToDevice);
  Seg X{dx, IN, 1, 1, 0, 0, IN, 0, B};
  GradMap gm{dg, flag, 0, (size_t)OUT * IN, 0, 0, OUT, IN};
  float* part; cudaMalloc(&part, (size_t)OUT * (IN + 1) * 4);
  const int direct = argc > 2 ? atoi(argv[2]) : 1;
  WgradArgs a{X, dd, OUT, OUT, IN, B, ((B + 31) / 32) * 32, part, gm, direct, 0, nullptr, nullptr, 0};
  using S = ws::MNShape<float, 128>;
  auto kern = ws::tc_mn_ws_kernel<float, 128>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
  dim3 grid((IN + 127) / 128, 1, 2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) kern<<<grid, ws::kThreads, S::SMEM>>>(a);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) kern<<<grid, ws::kThreads, S::SMEM>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("FC wgrad B=%d grid %dx%d stages=%d smem=%d: %.2f us/launch (%s)\n", B, grid.x, grid.z, S::NS, S::SMEM,
         ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  unsigned long long t[256];
  cudaMemcpyFromSymbol(t, g_trace, sizeof(t));
  printf("setup +%.0f\n", (double)(t[1] - t[0]));
  for (int i = 0; i < (B + 31) / 32; ++i)
    printf(" chunk %d: data +%.0f mma-ready +%.0f issued +%.0f\n", i, (double)(t[64 + 4 * i] - t[0]),
           (double)(t[8 + 2 * i] - t[0]), (double)(t[9 + 2 * i] - t[0]));
  printf("loop done +%.0f acc +%.0f stores +%.0f end +%.0f dealloc +%.0f\n", (double)(t[5] - t[0]), (double)(t[2] - t[0]),
         (double)(t[6] - t[0]), (double)(t[3] - t[0]), (double)(t[4] - t[0]));
  for (int c = 0; c < 4; ++c)
    printf("  epi iter %d: start +%.0f tmem +%.0f\n", c, (double)(t[100 + 2 * c] - t[0]), (double)(t[101 + 2 * c] - t[0]));
  return 0;
}
