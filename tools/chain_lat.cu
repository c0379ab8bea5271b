// chain_lat.cu -- dependent-kernel latency floor on B200 inside a CUDA graph:
// how long does a chain of N back-to-back kernels take per kernel, for
// kernels shaped like ours (grid, 288 threads, big dynamic smem, TMEM
// alloc, PDL)?  Debug tool, not product.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace ga3c;

__device__ float g_sink[1 << 20];

template <bool PDL, bool TMEM, bool TOUCH>
__global__ void k_chain(int iter) {
  extern __shared__ uint8_t sm[];
  __shared__ uint32_t tb;
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  if (TMEM && threadIdx.x >= 256) tc::tmem_alloc<64>(&tb);
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (TOUCH) {  // one dependent global round trip (read previous kernel's output)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    float v = g_sink[i & ((1 << 20) - 1)];
    g_sink[(i + 1) & ((1 << 20) - 1)] = v + 1.0f;
  }
  __syncthreads();
  if (TMEM && threadIdx.x >= 256) tc::tmem_dealloc<64>(tb);
}

template <bool PDL, bool TMEM, bool TOUCH>
float run(int grid, int smem, int n) {
  auto k = k_chain<PDL, TMEM, TOUCH>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n; ++i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(288);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = PDL ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, i);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / (10 * n);
}

int main() {
  const int n = 200;
  for (int grid : {1, 40, 148, 296}) {
    for (int smem : {0, 100 * 1024, 200 * 1024}) {
      printf("grid %3d smem %6d | plain %.2f us | pdl %.2f | pdl+tmem %.2f | pdl+tmem+touch %.2f | plain+touch %.2f\n",
             grid, smem, run<false, false, false>(grid, smem, n), run<true, false, false>(grid, smem, n),
             run<true, true, false>(grid, smem, n), run<true, true, true>(grid, smem, n),
             run<false, false, true>(grid, smem, n));
    }
  }
  return 0;
}
