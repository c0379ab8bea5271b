// tc_wgrad.cuh -- the MN-major GEMM contract (WgradArgs) and swizzle
// addressing for tc_ws.cuh's tc_mn_ws_kernel: weight gradients
// (nnet.cpp:58-73 summed over the batch, nnet.cpp:262-278)
//
//   dW[co][kk] = sum_m X(m, kk) * D(m, co)        db[co] = sum_m D(m, co)
//
// computed transposed as C'[kk][co] so the 128-lane MMA tile runs over the
// long kk axis and N = Cout, the reduction axis m (batch x output pixels)
// being the MMA K axis with both operands MN-major; and (mode 1) the FC input
// gradient dX^T = W^T dh^T with the lower layer's ReLU gate.  Split-K over
// blockIdx.y writes partials [split][Cout][Kw+1] (bias in the last column)
// that splitk_wgrad_kernel reduces in a fixed order.
#pragma once

#include <cstdint>

#include "gemm_simt.cuh"
#include "tc_common.cuh"
#include "tc_gemm.cuh"

namespace ga3c {

struct WgradArgs {
  Seg X;             // rows = pixels (M), k-runs along kk; X.rows = number of pixels
  const float* D;    // [pixels][ldd] output gradient (already ReLU-gated)
  int ldd;           // row stride of D
  int cout;          // N' (valid columns)
  int Kw;            // M' = kk extent (k*k*Cin or fan-in)
  int npix;          // reduction length
  int kc;            // pixels per split (multiple of 32)
  float* part;       // [split][cout][Kw+1]  (when !direct)
  GradMap gm;        // direct store (when splits == 1)
  int direct;
  // mode 1 (FC input gradient): out[co * ldo + kk] = gate[...] > 0 ? C' : 0,
  // no bias column; X = W rows (m = fan-out unit), D = dh^T [fan-out][batch]
  int mode;
  float* out;
  const float* gate;
  int ldo;
  // mode 0 with grid.y > 1 splits: reduce the partial tiles (and the bias
  // column) through DSMEM inside a (1, grid.y, 1) cluster and store dtheta
  // directly (no split-K partials, no reduction kernel)
  int cluster;
};

namespace detail {

// MN-major tf32 operands use SWIZZLE_128B_BASE32B (layout type 1): atoms of
// 4 k-rows x 128 B (32 MN elements), the 32-byte unit index XORed with
// row % 4.  Byte offset of 16-byte vector v (0..7) of MN atom g in k-row p
// (0..31 of the chunk): MN atoms are 512 B apart (LBO), 4-row k groups `sbo`
// apart (SBO).  Verified on B200 by tools/tc_probe.cu.
__device__ __forceinline__ uint32_t mn_off(int p, int g, int v, int sbo) {
  return static_cast<uint32_t>((p >> 2) * sbo + (g << 9) + ((p & 3) << 7) +
                               ((((v >> 1) ^ p) & 3) << 5) + ((v & 1) << 4));
}

}  // namespace detail

template <typename TX, int BN>
struct WgShape {
  static constexpr bool X_LO = sizeof(TX) == 4;
  static constexpr int A_BYTES = 32 * 128 * 4;  // 32 pixels x 128 kk fp32
  static constexpr int B_BYTES = 32 * BN * 4;   // 32 pixels x BN co fp32
  static constexpr int SBO_A = 4 * 512;         // 4 MN atoms of 32 kk per k group
  static constexpr int SBO_B = (BN / 32) * 512;
  static constexpr int STAGE = A_BYTES * (X_LO ? 2 : 1) + 2 * B_BYTES;
  static constexpr int SMEM = 2 * STAGE + 1024;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int BVEC = 32 * BN / 4;  // 16-byte vectors of the D tile
  static constexpr int BN_PER = (BVEC + kTcThreads - 1) / kTcThreads;
};

}  // namespace ga3c
