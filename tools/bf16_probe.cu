// bf16_probe.cu -- checks tc_u8_fwd_kernel (exact bf16 split of fp32 weights)
// against a CPU double reference on DNN A's conv1.  Debug tool, not product.
#include <cmath>
#include <cstring>
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>
#include "tc_bf16.cuh"
using namespace ga3c;

__global__ void write_frames(uint8_t* x, size_t n, int it) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = static_cast<uint8_t>((i * 2654435761u + it * 40503u) >> 13);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;  // 0 fp32 weights, 1 bf16-exact weights, 2 A=1 only
  const int ks = argc > 2 ? atoi(argv[2]) : 1;
  const int B = argc > 3 ? atoi(argv[3]) : 2, ih = 84, iw = 84, cin = 4, k = 8, s = 4, oh = 20, ow = 20, cout = 16, K = k * k * cin;
  std::mt19937 rng(5);
  std::vector<uint8_t> x(B * ih * iw * cin);
  for (auto& v : x) v = mode == 2 ? 1 : rng() & 255;
  std::vector<float> w(cout * K), b(cout, 0.0f);
  for (auto& v : w) {
    v = (rng() / 4294967296.0f - 0.5f) * 0.125f;
    if (mode == 1) {
      uint32_t u;
      memcpy(&u, &v, 4);
      u &= 0xFFFF0000u;
      memcpy(&v, &u, 4);
    }
  }
  uint8_t* dx; float *dw, *db, *dout;
  cudaMalloc(&dx, x.size()); cudaMalloc(&dw, w.size() * 4); cudaMalloc(&db, 64);
  const int M = B * oh * ow;
  cudaMalloc(&dout, (size_t)M * cout * 4);
  cudaMemcpy(dx, x.data(), x.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 64, cudaMemcpyHostToDevice);
  Seg A{dx, (long long)ih * iw * cin, oh * ow, ow, s * iw * cin, s * cin, k * cin, iw * cin, M};
  Seg W{dw, K, 1, 1, 0, 0, K, 0, cout};
  TcEpiArgs e{db, dout, cout};
  using S = bf::U8Shape<16>;
  auto kern = bf::tc_u8_fwd_kernel<16, false>;
  const int smem = S::NS_DEEP * S::STAGE + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kc = ((K / 64 + ks - 1) / ks) * 64;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((M + 127) / 128, ks, 1);
  cfg.blockDim = dim3(bf::kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = ks;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (argc > 4 && atoi(argv[4])) ? 2 : 1;
  const int iters = argc > 5 ? atoi(argv[5]) : 1;
  std::vector<float> out((size_t)M * cout);
  double worst_all = 0;
  cudaError_t err = cudaSuccess;
  for (int it = 0; it < iters; ++it) {
    if (iters > 1) {
      write_frames<<<64, 256>>>(dx, x.size(), it);
      cudaMemcpy(x.data(), dx, x.size(), cudaMemcpyDeviceToHost);
      write_frames<<<64, 256>>>(dx, x.size(), it);
    }
    cudaLaunchKernelEx(&cfg, kern, A, W, M, cout, K, kc, e);
    err = cudaDeviceSynchronize();
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int m = 0; m < M; ++m) {
      const int bb = m / (oh * ow), p = m % (oh * ow), oy = p / ow, ox = p % ow;
      for (int n = 0; n < cout; ++n) {
        double acc = 0;
        for (int ky = 0; ky < k; ++ky)
          for (int kx = 0; kx < k; ++kx)
            for (int c = 0; c < cin; ++c)
              acc += x[((size_t)(bb * ih + oy * s + ky) * iw + ox * s + kx) * cin + c] / 256.0 *
                     w[(size_t)n * K + (ky * k + kx) * cin + c];
        const double ref = acc < 0 ? 0 : acc;
        const double d = std::fabs(out[(size_t)m * cout + n] - ref);
        static int shown = 0;
        if (d > 1e-5 && shown < 12) {
          ++shown;
          printf("    m %d (tile %d row %d) n %d got %.6f ref %.6f\n", m, m / 128, m % 128, n,
                 out[(size_t)m * cout + n], ref);
        }
        worst = std::max(worst, d);
      }
    }
    worst_all = std::max(worst_all, worst);
    if (worst > 1e-5) printf("  iter %d: worst %.3e\n", it, worst);
  }
  printf("iters %d ks %d pdl %d: %s worst abs %.3e\n", iters, ks, (int)cfg.numAttrs - 1, cudaGetErrorString(err), worst_all);
  return 0;
}
