// tc_wgrad.cuh -- tcgen05 weight-gradient GEMM (nnet.cpp:58-73 summed over
// the batch, nnet.cpp:262-278), for conv (implicit im2col) and FC layers:
//
//   dW[co][kk] = sum_m X(m, kk) * D(m, co)        db[co] = sum_m D(m, co)
//
// computed transposed as C'[kk][co] so the 128-lane MMA tile runs over the
// long kk axis (k*k*Cin or the FC fan-in) and N = Cout.  The reduction axis m
// (batch x output pixels) is the MMA K axis; both operands are MN-major in
// memory (X rows and D rows are contiguous along kk / co), so they are staged
// in the 128B-swizzled MN-major canonical layout.  Split-K over blockIdx.y
// (fixed pixel ranges) writes partial sums [split][Cout][Kw+1] (bias in the
// last column, accumulated by the D-tile producers) that splitk_grad_kernel
// reduces in order; with one split the epilogue writes dtheta directly.
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

template <typename TX, int BN>
__global__ void __launch_bounds__(kTcThreads, 1) tc_wgrad_kernel(WgradArgs a) {
  static_assert(BN % 32 == 0, "MN-major SW128 needs 32-wide N atoms");
  using S = WgShape<TX, BN>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_red[4 * kTcThreads];  // [256 / (BN/4) rows][BN]
  uint8_t* smem = detail::align1024(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kk0 = blockIdx.x * 128;
  const int n0 = blockIdx.z * BN;
  const int split = blockIdx.y;
  const int pb = split * a.kc;
  const int pe = min(a.npix, pb + a.kc);
  const int nchunks = (pe - pb + 31) / 32;
  const bool do_bias = blockIdx.x == 0 && a.mode == 0;

  // X tile: thread -> (pixel row p, 16B vector v), 4 MN atoms g (kk chunks)
  const int xp = tid >> 3, xv = tid & 7;
  int xcoff[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int kk = kk0 + 32 * g;
    xcoff[g] = kk < a.Kw ? a.X.chunkoff(kk) : -1;
  }
  // D tile: idx = tid + 256 j -> (pixel p = idx / (BN/4), vector v = idx % (BN/4))
  constexpr int DV = BN / 4;
  float4 bsum[S::BN_PER];
#pragma unroll
  for (int j = 0; j < S::BN_PER; ++j) bsum[j] = make_float4(0.f, 0.f, 0.f, 0.f);

  // registers for one chunk
  float4 xr[4];
  uint32_t xw[4];
  float4 dr[S::BN_PER];
  auto load = [&](int c) {
    const int p0 = pb + 32 * c;
    const int pix = p0 + xp;
    const bool pv = pix < pe;
    const int rb = pv ? a.X.rowbase(pix) : 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const bool ok = pv && xcoff[g] >= 0;
      if constexpr (sizeof(TX) == 4) {
        xr[g] = ok ? __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(a.X.p) + rb +
                                                            xcoff[g]) + xv)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        xw[g] = ok ? __ldg(reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(a.X.p) + rb +
                                                              xcoff[g]) + xv)
                   : 0u;
      }
    }
#pragma unroll
    for (int j = 0; j < S::BN_PER; ++j) {
      const int idx = tid + kTcThreads * j;
      const int p = idx / DV, v = idx % DV;
      const int px = p0 + p;
      const int co = n0 + 4 * v;
      dr[j] = (idx < S::BVEC && px < pe && co < a.cout)
                  ? __ldg(reinterpret_cast<const float4*>(a.D + static_cast<std::size_t>(px) * a.ldd + co))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };

  if (nchunks > 0) load(0);
  if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t idesc = tc::idesc_tf32(128, BN, true, true);

  for (int i = 0; i < nchunks; ++i) {
    const int s = i & 1;
    if (i >= 2) tc::mbar_wait(&bars[s], ((i >> 1) - 1) & 1);
    const uint32_t st = tc::smem_u32(smem + s * S::STAGE);
    const uint32_t a_hi = st;
    const uint32_t a_lo = st + S::A_BYTES;
    const uint32_t b_hi = st + S::A_BYTES * (S::X_LO ? 2 : 1);
    const uint32_t b_lo = b_hi + S::B_BYTES;
    // X tile
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint32_t off = detail::mn_off(xp, g, xv, S::SBO_A);
      if constexpr (sizeof(TX) == 4) {
        float4 h, l;
        detail::split1(xr[g].x, h.x, l.x);
        detail::split1(xr[g].y, h.y, l.y);
        detail::split1(xr[g].z, h.z, l.z);
        detail::split1(xr[g].w, h.w, l.w);
        detail::sts128(a_hi + off, h);
        detail::sts128(a_lo + off, l);
      } else {
        float4 f;
        f.x = static_cast<float>(xw[g] & 0xFFu) * (1.0f / 256.0f);
        f.y = static_cast<float>((xw[g] >> 8) & 0xFFu) * (1.0f / 256.0f);
        f.z = static_cast<float>((xw[g] >> 16) & 0xFFu) * (1.0f / 256.0f);
        f.w = static_cast<float>(xw[g] >> 24) * (1.0f / 256.0f);
        detail::sts128(a_hi + off, f);
      }
    }
    // D tile (+ bias partial sums)
#pragma unroll
    for (int j = 0; j < S::BN_PER; ++j) {
      const int idx = tid + kTcThreads * j;
      if (idx >= S::BVEC) break;
      const int p = idx / DV, v = idx % DV;
      bsum[j].x += dr[j].x;
      bsum[j].y += dr[j].y;
      bsum[j].z += dr[j].z;
      bsum[j].w += dr[j].w;
      float4 h, l;
      detail::split1(dr[j].x, h.x, l.x);
      detail::split1(dr[j].y, h.y, l.y);
      detail::split1(dr[j].z, h.z, l.z);
      detail::split1(dr[j].w, h.w, l.w);
      const uint32_t off = detail::mn_off(p, v >> 3, v & 7, S::SBO_B);
      detail::sts128(b_hi + off, h);
      detail::sts128(b_lo + off, l);
    }
    if (i + 1 < nchunks) load(i + 1);
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // four 8-pixel k-steps = two 4-row k groups each
        const uint64_t dah = tc::sdesc(a_hi + 2 * h * S::SBO_A, 512, S::SBO_A, 1);
        const uint64_t dbh = tc::sdesc(b_hi + 2 * h * S::SBO_B, 512, S::SBO_B, 1);
        tc::mma_tf32(tmem, dah, dbh, idesc, (i | h) != 0);
        tc::mma_tf32(tmem, dah, tc::sdesc(b_lo + 2 * h * S::SBO_B, 512, S::SBO_B, 1), idesc, 1);
        if constexpr (S::X_LO)
          tc::mma_tf32(tmem, tc::sdesc(a_lo + 2 * h * S::SBO_A, 512, S::SBO_A, 1), dbh, idesc, 1);
      }
      tc::mma_commit(&bars[s]);
    }
  }

  const int last = nchunks - 1;
  if (nchunks > 0) {
    tc::mbar_wait(&bars[last & 1], (last >> 1) & 1);
  }
  tc::tc_fence_after();

  const int quad = warp & 3;
  const int row = quad * 32 + lane;
  const int kk = kk0 + row;
  constexpr int HALF = BN / 2;
  const int cbeg = (warp >> 2) * HALF;
  const int ldp = a.Kw + 1;
#pragma unroll
  for (int c = 0; c < HALF; c += 16) {
    const int c0 = cbeg + c;
    float v[16];
    if (nchunks > 0) {
      tc::tmem_ld16(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0, v);
      tc::tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
    }
    if (kk < a.Kw) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int co = n0 + c0 + j;
        if (co < a.cout) {
          if (a.mode == 1) {
            const std::size_t o = static_cast<std::size_t>(co) * a.ldo + kk;
            a.out[o] = __ldg(a.gate + o) <= 0.f ? 0.f : v[j];
          } else if (a.direct) {
            a.gm.store(co, kk, v[j]);
          } else {
            a.part[(static_cast<std::size_t>(split) * a.cout + co) * ldp + kk] = v[j];
          }
        }
      }
    }
  }
  if (do_bias) {
    // thread tid always owns columns 4*(tid % DV).. of pixel rows tid / DV
    // (+ 256/DV per pass): fold its passes, then sum the rows in order
    static_assert(kTcThreads % DV == 0, "BN must divide 1024");
    constexpr int R = kTcThreads / DV;
    float4 t = bsum[0];
#pragma unroll
    for (int j = 1; j < S::BN_PER; ++j) {
      t.x += bsum[j].x;
      t.y += bsum[j].y;
      t.z += bsum[j].z;
      t.w += bsum[j].w;
    }
    float* red = bias_red + (tid / DV) * BN + 4 * (tid % DV);
    red[0] = t.x;
    red[1] = t.y;
    red[2] = t.z;
    red[3] = t.w;
    __syncthreads();
    if (tid < BN) {
      float sacc = 0.f;
      for (int r = 0; r < R; ++r) sacc += bias_red[r * BN + tid];
      const int co = n0 + tid;
      if (co < a.cout) {
        if (a.direct)
          a.gm.store(co, a.Kw, sacc);
        else
          a.part[(static_cast<std::size_t>(split) * a.cout + co) * ldp + a.Kw] = sacc;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace ga3c
