// tc_trace.cu -- timeline of one CTA of the pipelined tcgen05 conv kernel
// (globaltimer at phase points).  Debug tool, not product.
#define GA3C_TRACE 1
#include <cstdio>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "tc_ws.cuh"
using namespace ga3c;

template <typename TA, int BN>
int run(int argc, char** argv);

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[2]) == "conv1") return run<uint8_t, 16>(argc, argv);
  return run<float, 32>(argc, argv);
}

template <typename TA, int BN>
int run(int argc, char** argv) {
  const bool c1 = sizeof(TA) == 1;
  const int B = argc > 1 ? atoi(argv[1]) : 40;
  // conv2 of DNN A: in [B][20][20][16] f32, W [32][4][4][16], out [B][9][9][32]
  const int ih = c1 ? 84 : 20, iw = ih, cin = c1 ? 4 : 16, k = c1 ? 8 : 4, s = c1 ? 4 : 2;
  const int oh = (ih - k) / s + 1, ow = oh, cout = c1 ? 16 : 32, K = k * k * cin;
  std::vector<TA> x(B * ih * iw * cin);
  std::vector<float> w(cout * K), b(cout, 0.01f);
  for (size_t i = 0; i < x.size(); ++i) x[i] = c1 ? (TA)((i * 7919) % 256) : (TA)((float)((i * 7919) % 1000) / 1000.f);
  for (size_t i = 0; i < w.size(); ++i) w[i] = (float)((i * 104729) % 1000) / 1000.f - 0.5f;
  TA* dx;
  float *dw, *db, *dout;
  cudaMalloc(&dx, x.size() * sizeof(TA)); cudaMalloc(&dw, w.size() * 4); cudaMalloc(&db, 128);
  cudaMalloc(&dout, (size_t)B * oh * ow * cout * 4);
  cudaMemcpy(dx, x.data(), x.size() * sizeof(TA), cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 128, cudaMemcpyHostToDevice);
  Seg A{dx, (long long)ih * iw * cin, oh * ow, ow, s * iw * cin, s * cin, k * cin, iw * cin, B * oh * ow};
  Seg W{dw, K, 1, 1, 0, 0, K, 0, cout};
  TcEpiArgs e{db, dout, cout};
  using S = ws::KKShape<TA, float, BN>;
  auto kern = ws::tc_kk_ws_kernel<TA, float, BN, TC_EPI_BIAS_RELU>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
  const int M = B * oh * ow;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) kern<<<(M + 127) / 128, ws::kThreads, S::SMEM>>>(A, W, M, cout, K, K, e);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) kern<<<(M + 127) / 128, ws::kThreads, S::SMEM>>>(A, W, M, cout, K, K, e);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  {  // same with programmatic dependent launch, eager and in a graph
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((M + 127) / 128); cfg.blockDim = dim3(ws::kThreads); cfg.dynamicSmemBytes = S::SMEM;
    cudaStream_t st; cudaStreamCreate(&st); cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int pdl = 0; pdl < 2; ++pdl) {
      cfg.numAttrs = pdl;
      for (int it = 0; it < 5; ++it) cudaLaunchKernelEx(&cfg, kern, A, W, M, cout, K, K, e);
      cudaEventRecord(e0, st);
      for (int it = 0; it < 20; ++it) cudaLaunchKernelEx(&cfg, kern, A, W, M, cout, K, K, e);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float m2; cudaEventElapsedTime(&m2, e0, e1);
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int it = 0; it < 20; ++it) cudaLaunchKernelEx(&cfg, kern, A, W, M, cout, K, K, e);
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e0, st);
      for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float m3; cudaEventElapsedTime(&m3, e0, e1);
      printf("pdl=%d: eager %.2f us/launch, graph %.2f us/launch (%s)\n", pdl, m2 * 1000 / 20, m3 * 1000 / 100,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  printf("B=%d M=%d CTAs=%d stages=%d smem=%d: %.2f us/launch (%s)\n", B, M, (M + 127) / 128, S::NS, S::SMEM,
         ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  unsigned long long t[256];
  cudaMemcpyFromSymbol(t, g_trace, sizeof(t));
  printf("setup %.0f ns, producers done +%.0f\n", (double)(t[1] - t[0]), (double)(t[5] - t[0]));
  for (int i = 0; i < K / 32; ++i)
    printf(" chunk %d: data(p0) +%.0f  mma-ready +%.0f  mma-issued +%.0f\n", i, (double)(t[64 + 4 * i] - t[0]),
           (double)(t[8 + 2 * i] - t[0]), (double)(t[9 + 2 * i] - t[0]));
  printf("mma done +%.0f, epilogue done +%.0f, dealloc +%.0f\n", (double)(t[2] - t[0]), (double)(t[3] - t[0]),
         (double)(t[4] - t[0]));
  return 0;
}
