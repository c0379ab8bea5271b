// mma_rate.cu -- tcgen05.mma kind::tf32 issue/throughput vs N (M=128, K=8),
// single CTA, operands in smem.  Debug tool, not product.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace ga3c;

template <int N>
__global__ void rate(int iters, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sa[16384];
  __shared__ __align__(1024) uint8_t sb[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(sa)[i] = 0.5f;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(sb)[i] = 0.25f;
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tb);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, N, false, false);
    const uint64_t da = tc::sdesc_sw128(tc::smem_u32(sa), 16, 1024);
    const uint64_t db = tc::sdesc_sw128(tc::smem_u32(sb), 16, 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) tc::mma_tf32(tb, da + 2 * (i & 3), db + 2 * (i & 3), idesc, i > 0);
    unsigned long long t1 = clock64();
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tb);
}

template <int N>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  unsigned long long h[2];
  for (int iters : {12, 96, 960}) {
    rate<N><<<1, 128>>>(iters, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d iters=%4d: issue %6llu cyc (%.1f/mma), complete %6llu cyc (%.1f/mma) -> %.0f MAC/clk\n", N, iters,
           h[0], (double)h[0] / iters, h[1], (double)h[1] / iters, 128.0 * N * 8 * iters / h[1]);
  }
}

int main() {
  run<16>(); run<32>(); run<64>(); run<128>(); run<256>();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
