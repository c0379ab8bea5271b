// tc_peak.cu -- measured dense tcgen05 peaks per MMA kind on this B200
// (kind::tf32, kind::f16 with bf16 operands, kind::i8), the denominators of
// the per-precision tensor fractions bench.py reports.  One CTA per SM, one
// elected thread issuing M=128 x N=256 MMAs back to back from smem operands
// into a TMEM accumulator, timed with CUDA events over the whole grid.
// Probe tool, not product.  Output: one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1611_06256_b200/csrc tools/tc_peak.cu -o tools/tc_peak
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"
#include "tc_pipe.cuh"
#include "tc_ws.cuh"
#include "tc_bf16.cuh"
#include "tc_u8conv.cuh"

using namespace ga3c;

constexpr int kM = 128, kN = 256;

// kind: 0 = tf32 (K = 8 per MMA), 1 = bf16 (K = 16), 2 = i8 (K = 32)
template <int KIND>
__global__ void __launch_bounds__(128) peak_kernel(int iters, int* sink) {
  __shared__ __align__(1024) uint8_t sb[kN * 128];
  uint8_t* sa = sb;  // operand values do not matter; A aliases B's first 128 rows
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
    for (int i = threadIdx.x; i < (int)sizeof(sb) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tb);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    // K-major SWIZZLE_128B tiles: 8-row groups 1024 B apart, one 128-byte
    // K chunk per MMA (tf32 8 x 4 B, bf16 16 x 2 B, i8 32 x 1 B)
    const uint64_t da = tc::sdesc_sw128(tc::smem_u32(sa), 16, 1024);
    const uint64_t db = tc::sdesc_sw128(tc::smem_u32(sb), 16, 1024);
    for (int i = 0; i < iters; ++i) {
      if constexpr (KIND == 0)
        tc::mma_tf32(tb, da, db, tc::idesc_tf32(kM, kN, false, false), i > 0);
      else if constexpr (KIND == 1)
        bf::mma_bf16(tb, da, db, bf::idesc_bf16(kM, kN), i > 0);
      else
        u8c::mma_i8(tb, da, db, u8c::idesc_u8s8(kM, kN), i > 0);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0 && iters < 0) *sink = 1;
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tb);
}

template <int KIND>
double measure(int sms, int iters) {
  int* sink;
  cudaMalloc(&sink, 4);
  peak_kernel<KIND><<<sms, 128>>>(iters / 10, sink);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    peak_kernel<KIND><<<sms, 128>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const int K = KIND == 0 ? 8 : KIND == 1 ? 16 : 32;
    const double ops = 2.0 * kM * kN * K * (double)iters * sms;
    best = ops / (ms * 1e-3) / 1e12 > best ? ops / (ms * 1e-3) / 1e12 : best;
  }
  cudaFree(sink);
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 200000;
  const double tf32 = measure<0>(sms, iters);
  const double bf16 = measure<1>(sms, iters);
  const double i8 = measure<2>(sms, iters);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"tf32_tflops\": %.1f, \"bf16_tflops\": %.1f, \"i8_tops\": %.1f, \"sms\": %d, \"mma\": \"M=%d N=%d "
         "cta_group::1, one CTA per SM\", \"max_sm_clock_mhz\": %d, \"error\": \"%s\"}\n",
         tf32, bf16, i8, sms, kM, kN, clk / 1000, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
