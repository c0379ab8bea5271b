// heads_trace.cu -- phase timeline of heads_loss_kernel (CTA 0, globaltimer).
// Debug tool, not product: compiles kernels.cu with GA3C_HTRACE.
#define GA3C_HTRACE 1
#include "../paper_1611_06256_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
using namespace ga3c;

int main() {
  const int B = 40, D = 256, A = 6, S = 41;
  std::vector<float> part((size_t)S * B * D), theta(D * (A + 1) + A + 1 + D), bias(D, 0.01f);
  for (size_t i = 0; i < part.size(); ++i) part[i] = ((i * 7919) % 1000) / 1000.f - 0.45f;
  for (size_t i = 0; i < theta.size(); ++i) theta[i] = ((i * 104729) % 1000) / 1000.f - 0.5f;
  std::vector<int> act(B);
  std::vector<double> ret(B);
  for (int b = 0; b < B; ++b) { act[b] = b % A; ret[b] = 0.1 * b - 2; }
  float *dp, *dth, *db, *dh_io, *dv, *dhead, *dh, *dhT; double *dpi, *dret, *dscal, *dsum; int *dact, *flag;
  unsigned* ticket;
  cudaMalloc(&dp, part.size() * 4); cudaMalloc(&dth, theta.size() * 4); cudaMalloc(&db, D * 4);
  cudaMalloc(&dh_io, B * D * 4); cudaMalloc(&dv, B * 4); cudaMalloc(&dhead, B * (A + 1) * 4);
  cudaMalloc(&dh, B * D * 4); cudaMalloc(&dhT, D * 64 * 4); cudaMalloc(&dpi, B * A * 8);
  cudaMalloc(&dret, B * 8); cudaMalloc(&dscal, B * 24); cudaMalloc(&dsum, 24); cudaMalloc(&dact, B * 4);
  cudaMalloc(&flag, 4); cudaMalloc(&ticket, 4); cudaMemset(ticket, 0, 4);
  cudaMemcpy(dp, part.data(), part.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dth, theta.data(), theta.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bias.data(), D * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dact, act.data(), B * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dret, ret.data(), B * 8, cudaMemcpyHostToDevice);
  const size_t smem = ((size_t)D * (A + 2) + 8 * (A + 1)) * 4;
  cudaFuncSetAttribute(heads_loss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 30; ++it) {
    if (it == 10) cudaEventRecord(e0);
    heads_loss_kernel<<<B, 256, smem>>>(dp, S, db, dh_io, B, D, dth, 0, (size_t)A * D, (size_t)A * D + A,
                                        (size_t)A * D + A + D, A, dact, dret, 0.01, 1e-6, 0.5, dpi, dv, dhead, dh,
                                        dhT, 64, dscal, flag);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long t[32];
  cudaMemcpyFromSymbol(t, g_htrace, sizeof(t));
  printf("heads_loss B=%d S=%d: %.2f us/launch (%s)\n", B, S, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  const char* nm[] = {"start", "w_issue", "partials", "w_wait", "logits", "softmax", "loss", "dh", "ticket", "end"};
  for (int i = 1; i < 10; ++i) printf("  %-9s +%6.0f ns\n", nm[i], (double)(t[i] - t[0]));
  return 0;
}
