// tma_probe.cu -- throughput of TMA im2col loads vs tiled loads of the same
// bytes (large s1 conv2 forward geometry: NHWC fp32 input [B][77][77][32],
// 4x4 window, stride 2, 128 output pixels x 32 channels per box).  One CTA
// per SM, one thread keeps an NS-deep ring of 16 KB boxes in flight, nothing
// consumes them: the rate is the TMA + L2/HBM path alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../include -I../paper_1611_06256_b200/csrc tma_probe.cu -o tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "tc_common.cuh"
#include "tc_gemm.cuh"

using namespace ga3c;

constexpr int NS = 8;
constexpr int BOX = 128 * 128;

__global__ void __launch_bounds__(32, 1) probe(const __grid_constant__ TmaConv tm, int mode, int ntiles, int P,
                                               int ow, int nk) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[NS];
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t base = tc::smem_u32(smem);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NS; ++s) tc::mbar_init(&full[s], 1);
  tc::fence_barrier_init();
  int n = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int m0 = t * 128;
    const int img = m0 / P, pp = m0 - img * P, oy = pp / ow;
    const int w0 = (pp - oy * ow) * 2, h0 = oy * 2;
    for (int c = 0; c < nk; ++c, ++n) {
      const int s = n % NS;
      if (n >= NS) tc::mbar_wait(&full[s], ((n / NS) - 1) & 1);
      tc::mbar_expect_tx(&full[s], BOX);
      if (mode == 0) {
        const int tap = c, ky = tap / 4, kx = tap % 4;
        tc::tma_im2col_4d(base + s * BOX, &tm.a, 0, w0, h0, img, static_cast<uint16_t>(kx),
                          static_cast<uint16_t>(ky), &full[s]);
      } else {
        // the same number of bytes as contiguous 128-pixel x 32-channel boxes
        tc::tma_tile_2d(base + s * BOX, &tm.b, 0, (m0 + 128 * c) % (P * 1024 - 128), &full[s]);
      }
    }
  }
  for (int k = n; k < n + NS; ++k)
    if (k >= NS) tc::mbar_wait(&full[k % NS], ((k / NS) - 1) & 1);
}

int main() {
  const int B = 1024, IH = 77, IW = 77, C = 32, OH = 37, OW = 37;
  const size_t bytes = size_t(B) * IH * IW * C * 4;
  float* x = nullptr;
  if (cudaMalloc(&x, bytes) != cudaSuccess) return 1;
  cudaMemset(x, 0, bytes);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q);
  auto enc_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col>(f);
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(f);
  TmaConv tm{};
  const cuuint64_t gdim[4] = {C, IW, IH, B};
  const cuuint64_t gstr[3] = {C * 4ull, IW * C * 4ull, size_t(IH) * IW * C * 4};
  const int lower[2] = {0, 0}, upper[2] = {-3, -3};
  const cuuint32_t es[4] = {1, 2, 2, 1};
  CUresult r1 = enc_im2col(&tm.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, gdim, gstr, lower, upper, 32, 128, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const cuuint64_t tdim[2] = {C, cuuint64_t(B) * IH * IW};
  const cuuint64_t tstr[1] = {C * 4ull};
  const cuuint32_t box[2] = {32, 128}, one[2] = {1, 1};
  CUresult r2 = enc_tiled(&tm.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, tdim, tstr, box, one,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
    printf("encode failed %d %d\n", r1, r2);
    return 1;
  }
  const int P = OH * OW, ntiles = (B * P + 127) / 128, nk = 16;
  const int smem = NS * BOX + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      probe<<<148, 32, smem>>>(tm, mode, ntiles, P, OW, nk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gb = double(ntiles) * nk * BOX / 1e9;
      printf("%s: %.1f us, %.2f GB loaded, %.2f TB/s (%s)\n", mode == 0 ? "im2col" : "tiled ", ms * 1e3, gb,
             gb / (ms * 1e-3) / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
