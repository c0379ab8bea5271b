// tc_gemm.cuh -- operand addressing shared by the tcgen05 GEMMs (tc_ws.cuh,
// tc_bf16.cuh, tc_u8conv.cuh, tc_dgrad.cuh):
//
//   Seg        row r / k-chunk k0 -> element offset of a contiguous run of
//              k elements: the implicit im2col of an NHWC activation or u8
//              frame (r = (b, oy, ox), k = (ky, kx, ci)) or a dense matrix
//   TcEpiArgs  the K-major GEMMs' epilogue contract (bias + ReLU rows, or
//              transposed split-K partials)
//   detail::   shared-memory stores and alignment helpers
#pragma once

#include <cuda.h>

#include <cstdint>

#include "tc_common.cuh"

namespace ga3c {

constexpr int kTcThreads = 256;

// Row r / k-chunk start k0 -> element offset of 32 contiguous elements.
//   conv (im2col): r = (b, oy, ox), k = (ky, kx, ci), run = k*cin
//   dense rows   : P = ow = 1, bstride = ld, rowlen = K
// Offsets must fit in 31 bits (checked by the dispatcher).
struct Seg {
  const void* p;
  long long bstride;
  int P, ow, rs_y, rs_x;  // rs_y = stride*iw*cin, rs_x = stride*cin
  int rowlen, kstride;    // contiguous run along k, stride between runs
  int rows;               // valid rows
  __device__ __forceinline__ int rowbase(int r) const {
    const int b = r / P;
    const int pp = r - b * P;
    const int oy = pp / ow;
    const int ox = pp - oy * ow;
    return static_cast<int>(b * bstride) + oy * rs_y + ox * rs_x;
  }
  __device__ __forceinline__ int chunkoff(int k0) const {
    const int ky = k0 / rowlen;
    return ky * kstride + (k0 - ky * rowlen);
  }
};

enum { TC_EPI_BIAS_RELU = 0, TC_EPI_PART_T = 1 };

// TMA-staged conv forward operands (tc_kk_ws_kernel<float, float, BN, 0, CAP,
// true>): `a` is an im2col tensor map over the NHWC fp32 input [B][IH][IW][Cin]
// (Cin % 32 == 0; 32 channels x 128 output pixels per box, traversal stride
// = the conv stride, bounding box = the VALID window range), `b` a tiled map
// over the OHWI weights [Cout][k*k*Cin] (box 32 x BN); both SWIZZLE_128B,
// i.e. exactly the K-major canonical layout the tf32 MMA descriptors read.
struct alignas(64) TmaConv {
  CUtensorMap a;
  CUtensorMap b;
  int cin, k, stride;
};

struct TcEpiArgs {
  const float* bias;  // per n (TC_EPI_BIAS_RELU)
  float* out;
  int ldo;  // BIAS_RELU: row stride of out;  PART_T: M (out is [split][N][M])
};

namespace detail {

__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}


__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  return reinterpret_cast<uint8_t*>((a + 1023) & ~static_cast<uintptr_t>(1023));
}

}  // namespace detail

template <typename TA, typename TB, int BN>
struct TcShape {
  static constexpr bool A_LO = sizeof(TA) == 4;
  static constexpr bool B_LO = sizeof(TB) == 4;
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE = A_BYTES * (A_LO ? 2 : 1) + B_BYTES * (B_LO ? 2 : 1);
  static constexpr int SMEM = 2 * STAGE + 1024;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

}  // namespace ga3c
