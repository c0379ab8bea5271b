// gemm_simt.cuh -- operand loaders, epilogues and the generic fp32 SIMT
// implicit-GEMM kernel used for every contraction of the GA3C trunk:
//   C[m][n] = sum_k A(m,k) * B(n,k)
// A and B are described by loader functors (dense row-major, transposed, or
// an on-the-fly NHWC im2col gather), so conv forward, conv weight-gradient,
// FC forward/dgrad/wgrad and the heads weight-gradient are all instances of
// one kernel with different loaders/epilogues.  Split-K partials are reduced
// in a fixed order by a second kernel, so every result is deterministic
// (no float atomics; SURVEY.md §7 "Determinism").
#pragma once

#include <cstdint>

#include "pdl.cuh"

namespace ga3c {

// ------------------------------------------------------------ loaders
// load(i, k): i indexes M (for A) or N (for B); K_CONTIG says which index is
// contiguous in memory so the tile loader can coalesce.

struct DenseK {  // X[i][k] row-major, k contiguous
  const float* p;
  int ld;
  static constexpr bool K_CONTIG = true;
  __device__ __forceinline__ float operator()(int i, int k) const {
    return __ldg(p + static_cast<std::size_t>(i) * ld + k);
  }
};

template <typename T>
struct DenseKIn {  // network input rows (u8 frames scaled by 1/256, or f32)
  const T* p;
  int ld;
  static constexpr bool K_CONTIG = true;
  __device__ __forceinline__ float operator()(int i, int k) const {
    if constexpr (sizeof(T) == 1)
      return static_cast<float>(p[static_cast<std::size_t>(i) * ld + k]) * (1.0f / 256.0f);
    else
      return __ldg(reinterpret_cast<const float*>(p) + static_cast<std::size_t>(i) * ld + k);
  }
};

struct DenseT {  // element (i, k) at p[k*ld + i], i contiguous
  const float* p;
  int ld;
  static constexpr bool K_CONTIG = false;
  __device__ __forceinline__ float operator()(int i, int k) const {
    return __ldg(p + static_cast<std::size_t>(k) * ld + i);
  }
};

template <typename T>
struct DenseTIn {  // network input, transposed view (i = feature, k = sample)
  const T* p;
  int ld;
  static constexpr bool K_CONTIG = false;
  __device__ __forceinline__ float operator()(int i, int k) const {
    if constexpr (sizeof(T) == 1)
      return static_cast<float>(p[static_cast<std::size_t>(k) * ld + i]) * (1.0f / 256.0f);
    else
      return __ldg(reinterpret_cast<const float*>(p) + static_cast<std::size_t>(k) * ld + i);
  }
};

// NHWC im2col of a VALID conv: row r = (b, oy, ox), column c = (ky, kx, ci).
template <typename T>
struct Im2col {
  const T* p;
  int ih, iw, cin, stride, ow, P, rowlen;  // rowlen = k*cin
  long long bstride;                      // elements between consecutive images
  __device__ __forceinline__ float at(int r, int c) const {
    const int b = r / P;
    const int pp = r - b * P;
    const int oy = pp / ow;
    const int ox = pp - oy * ow;
    const int ky = c / rowlen;
    const int rr = c - ky * rowlen;
    const std::size_t idx = static_cast<std::size_t>(b) * bstride +
        (static_cast<std::size_t>(oy * stride + ky) * iw + ox * stride) * cin + rr;
    if constexpr (sizeof(T) == 1)
      return static_cast<float>(p[idx]) * (1.0f / 256.0f);
    else
      return __ldg(reinterpret_cast<const float*>(p) + idx);
  }
};

template <typename T>
struct Im2colA : Im2col<T> {  // A(m = r, k = c)
  static constexpr bool K_CONTIG = true;
  __device__ __forceinline__ float operator()(int i, int k) const { return this->at(i, k); }
};

template <typename T>
struct Im2colB : Im2col<T> {  // B(n = c, k = r): weight-gradient operand
  static constexpr bool K_CONTIG = false;
  __device__ __forceinline__ float operator()(int i, int k) const { return this->at(k, i); }
};

// Appends a column of ones at i == n_real: the GEMM then also produces the
// bias gradient sum_k A(m,k) in column n_real.
template <typename L>
struct WithOnes {
  L l;
  int n_real;
  static constexpr bool K_CONTIG = L::K_CONTIG;
  __device__ __forceinline__ float operator()(int i, int k) const {
    return i == n_real ? 1.0f : l(i, k);
  }
};

// ---------------------------------------------------------- epilogues

struct EpiBiasRelu {  // out[m][n] = max(acc + bias[n], 0)  (nnet.cpp:99)
  float* out;
  const float* bias;
  int ldo;
  __device__ __forceinline__ void operator()(int m, int n, float acc, int) const {
    float v = acc + __ldg(bias + n);
    out[static_cast<std::size_t>(m) * ldo + n] = v < 0.0f ? 0.0f : v;
  }
};

struct EpiPartial {  // split-K partial sums, reduced later in a fixed order
  float* part;
  int M, N;
  __device__ __forceinline__ void operator()(int m, int n, float acc, int split) const {
    part[(static_cast<std::size_t>(split) * M + m) * N + n] = acc;
  }
};

struct EpiGate {  // out = gate > 0 ? acc : 0   (ReLU gate, nnet.cpp:268-270)
  float* out;
  const float* gate;
  int ldo;
  __device__ __forceinline__ void operator()(int m, int n, float acc, int) const {
    const std::size_t i = static_cast<std::size_t>(m) * ldo + n;
    out[i] = __ldg(gate + i) <= 0.0f ? 0.0f : acc;
  }
};

// Row m of a weight-gradient GEMM [rows][Kw+1] -> flat dtheta offsets.
// Rows [0, rows0) map to (w0, b0); the rest to (w1, b1) (used by the heads:
// policy rows then the value row).  Sets *flag on any non-finite component
// (consumed by rmsprop, nnet.cpp:299-301).
struct GradMap {
  float* dtheta;
  int* flag;
  std::size_t w0, b0, w1, b1;
  int rows0, Kw;
  __device__ __forceinline__ void store(int m, int n, float v) const {
    std::size_t idx;
    const bool first = m < rows0;
    const int mm = first ? m : m - rows0;
    if (n < Kw)
      idx = (first ? w0 : w1) + static_cast<std::size_t>(mm) * Kw + n;
    else
      idx = (first ? b0 : b1) + mm;
    dtheta[idx] = v;
    if (!isfinite(v)) atomicOr(flag, 1);
  }
};

struct EpiGrad {
  GradMap g;
  __device__ __forceinline__ void operator()(int m, int n, float acc, int) const {
    g.store(m, n, acc);
  }
};

// ------------------------------------------------------------- kernel

constexpr int kBM = 64, kBN = 64, kBK = 16, kThreads = 256;

template <class LA, class LB, class Epi>
__global__ void __launch_bounds__(kThreads)
gemm_simt_kernel(LA la, LB lb, Epi epi, int M, int N, int K, int k_chunk) {
  pdl_enter();
  __shared__ __align__(16) float As[2][kBK][kBM + 4];
  __shared__ __align__(16) float Bs[2][kBK][kBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  const int split = blockIdx.z;
  const int kb = split * k_chunk;
  const int ke = min(K, kb + k_chunk);

  float ra[4], rb[4];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int mi, ki;
      if constexpr (LA::K_CONTIG) {
        ki = tid & (kBK - 1);
        mi = (tid >> 4) + j * (kThreads / kBK);
      } else {
        mi = tid & (kBM - 1);
        ki = (tid >> 6) + j * (kThreads / kBM);
      }
      const int gm = m0 + mi, gk = k0 + ki;
      ra[j] = (gm < M && gk < ke) ? la(gm, gk) : 0.0f;
      int ni, kj;
      if constexpr (LB::K_CONTIG) {
        kj = tid & (kBK - 1);
        ni = (tid >> 4) + j * (kThreads / kBK);
      } else {
        ni = tid & (kBN - 1);
        kj = (tid >> 6) + j * (kThreads / kBN);
      }
      const int gn = n0 + ni, gk2 = k0 + kj;
      rb[j] = (gn < N && gk2 < ke) ? lb(gn, gk2) : 0.0f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int mi, ki;
      if constexpr (LA::K_CONTIG) {
        ki = tid & (kBK - 1);
        mi = (tid >> 4) + j * (kThreads / kBK);
      } else {
        mi = tid & (kBM - 1);
        ki = (tid >> 6) + j * (kThreads / kBM);
      }
      As[buf][ki][mi] = ra[j];
      int ni, kj;
      if constexpr (LB::K_CONTIG) {
        kj = tid & (kBK - 1);
        ni = (tid >> 4) + j * (kThreads / kBK);
      } else {
        ni = tid & (kBN - 1);
        kj = (tid >> 6) + j * (kThreads / kBN);
      }
      Bs[buf][kj][ni] = rb[j];
    }
  };

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  int buf = 0;
  if (kb < ke) {
    load_tile(kb);
    store_tile(0);
  }
  __syncthreads();
  for (int k0 = kb; k0 < ke; k0 += kBK) {
    const bool more = k0 + kBK < ke;
    if (more) load_tile(k0 + kBK);
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) store_tile(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < N) epi(m, n, acc[i][j], split);
    }
  }
}

}  // namespace ga3c
