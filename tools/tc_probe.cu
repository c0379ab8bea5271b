// tc_probe.cu -- hardware probe for tcgen05 kind::tf32 shared-memory
// operand layouts (K-major vs MN-major, SW128).  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_1611_06256_b200/csrc tc_probe.cu -o tc_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace ga3c;

// A: M=128 x K=8, B: N=32 x K=8.  mode bit0: A MN-major, bit1: B MN-major.
__global__ void probe(const float* A, const float* B, float* C, int mode, int lbo_a, int sbo_a,
                      int lbo_b, int sbo_b) {
  __shared__ __align__(1024) uint8_t sa[20480];
  __shared__ __align__(1024) uint8_t sb[8192];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  // zero
  for (int i = tid; i < (int)sizeof(sa) / 4; i += blockDim.x) reinterpret_cast<float*>(sa)[i] = 0.f;
  for (int i = tid; i < (int)sizeof(sb) / 4; i += blockDim.x) reinterpret_cast<float*>(sb)[i] = 0.f;
  __syncthreads();
  float* fa = reinterpret_cast<float*>(sa);
  float* fb = reinterpret_cast<float*>(sb);
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    uint32_t off;
    if (mode & 1) {  // MN-major SW128_32B: atom (g = m/32, h = k/4) 4 rows x 128 B
      const int g = m / 32, h = k / 4, r = k % 4, c = (m % 32) / 8, e = m % 8;
      off = g * lbo_a + h * sbo_a + r * 128 + (((c ^ r) & 3) << 5) + e * 4;
    } else {  // K-major: row m, k chunk (k/4) of a 128B row (only first 32B used)
      off = tc::sw128_off(m, k / 4) + (k % 4) * 4;
    }
    fa[off / 4] = A[m * 8 + k];
  }
  for (int i = tid; i < 32 * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8;
    uint32_t off;
    if (mode & 2) {
      const int h = k / 4, r = k % 4, c = n / 8, e = n % 8;
      off = h * sbo_b + r * 128 + (((c ^ r) & 3) << 5) + e * 4;
    } else {
      off = tc::sw128_off(n, k / 4) + (k % 4) * 4;
    }
    fb[off / 4] = B[n * 8 + k];
  }
  if (threadIdx.x < 32) tc::tmem_alloc<32>(&tbase);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, 32, mode & 1, (mode & 2) != 0);
    uint64_t da = (mode & 1) ? tc::sdesc(tc::smem_u32(sa), lbo_a, sbo_a, 1)
                             : tc::sdesc_sw128(tc::smem_u32(sa), 16, 1024);
    uint64_t db = (mode & 2) ? tc::sdesc(tc::smem_u32(sb), lbo_b, sbo_b, 1)
                             : tc::sdesc_sw128(tc::smem_u32(sb), 16, 1024);
    tc::mma_tf32(tm, da, db, idesc, 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < 32; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tm + ((warp * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) C[(warp * 32 + lane) * 32 + c0 + j] = v[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<32>(tm);
}

int main() {
  float hA[128 * 8], hB[32 * 8], ref[128 * 32], hC[128 * 32];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 37) % 17 - 8);
  for (int i = 0; i < 32 * 8; ++i) hB[i] = (float)((i * 11) % 13 - 6);
  {  // tf32 operand conversion: truncation or rounding?  x = 1 + 0.75 ulp(tf32)
    float *dA, *dB, *dC;
    float a[128 * 8] = {0}, b[32 * 8] = {0}, c[128 * 32];
    a[0] = 1.0f + 0x1.0p-11f + 0x1.0p-12f;  // A[0][0]
    b[0] = 1.0f;                            // B[0][0]
    cudaMalloc(&dA, sizeof(a)); cudaMalloc(&dB, sizeof(b)); cudaMalloc(&dC, sizeof(c));
    cudaMemcpy(dA, a, sizeof(a), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, b, sizeof(b), cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, dC, 0, 0, 0, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(c, dC, sizeof(c), cudaMemcpyDeviceToHost);
    printf("tf32 conversion probe: x=%.9g -> C=%.9g (trunc 1.0, RN %.9g)\n", a[0], c[0], 1.0 + 0x1.0p-10);
  }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      float s = 0;
      for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[n * 8 + k];
      ref[m * 32 + n] = s;
    }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dC, sizeof(hC));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  struct Cfg { int mode, la, sa, lb, sb; } cfgs[] = {
      {0, 0, 0, 0, 0},          {1, 512, 2048, 0, 0}, {1, 1024, 512, 0, 0},
      {2, 0, 0, 512, 512},      {2, 0, 0, 4096, 512},  {3, 512, 2048, 512, 512},
      {3, 1024, 512, 4096, 512}, {1, 2048, 512, 0, 0}, {2, 0, 0, 512, 1024}, {1, 512, 4096, 0, 0}};
  for (auto& c : cfgs) {
    cudaMemset(dC, 0, sizeof(hC));
    probe<<<1, 128>>>(dA, dB, dC, c.mode, c.la, c.sa, c.lb, c.sb);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hC, dC, sizeof(hC), cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int i = 0; i < 128 * 32; ++i) {
      err += (hC[i] - ref[i]) * (double)(hC[i] - ref[i]);
      nrm += ref[i] * (double)ref[i];
    }
    printf("mode %d lboA %5d sboA %5d lboB %5d sboB %5d : %s rel_err %.3e  C[0]=%g ref %g C[33*32+5]=%g ref %g\n",
           c.mode, c.la, c.sa, c.lb, c.sb, cudaGetErrorString(e), err / (nrm + 1e-30), hC[0], ref[0],
           hC[33 * 32 + 5], ref[33 * 32 + 5]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
