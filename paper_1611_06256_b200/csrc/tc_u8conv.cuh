// tc_u8conv.cuh -- persistent, weight-stationary conv forward on raw u8
// frames with tcgen05.mma kind::i8 (u8 x s8 -> exact s32 accumulate).
//
// Arithmetic (nnet.cpp:91-119 forward, conv layer 0, restated):
//   * the frame bytes x are the A operand as they are (u8, the 1/256 input
//     scale is a power of two applied in the epilogue);
//   * each output channel's fp32 weights are put on a per-channel power-of-two
//     grid, q = rn(w * 2^(30-e_n)) with 2^e_n > max|w_n|, so |q| <= 2^30 and
//     |q - w 2^(30-e_n)| <= 1/2 (weights within 2^-31 max|w_n| -- below fp32's
//     own 2^-24 relative rounding), and q is split exactly into four signed
//     byte digits, q = d0 2^24 + d1 2^16 + d2 2^8 + d3;
//   * the four digit rows are N-concatenated ([d0; d1; d2; d3], N = 4*BN) so
//     one MMA per 32-wide k step produces all four exact s32 dot products;
//   * the epilogue converts the four exact s32 sums to fp32 and combines them
//     smallest first (d3 + 2^8 d2 + 2^16 d1 + 2^24 d0: three roundings), then
//     applies the power-of-two scale 2^(e_n-38) and the bias in one FMA.
// The result is fp32-accurate (weights within 2^-31 max|w_n|, a few fp32
// roundings in the combination, none in the 256-term dot products), at half
// the MMA cost of tc_bf16.cuh's three bf16 pieces (int8 runs at twice the
// bf16 rate) and with no u8 -> bf16 conversion in the mainloop.
//
// Data movement:
//   * W is quantized and laid out in shared memory ONCE per CTA;
//   * each 128-pixel tile's input footprint -- rows oy*s .. oy*s+k-1 of the
//     (at most two) frames the tile touches, one contiguous byte range per
//     frame -- arrives by 1-D TMA bulk copy (cp.async.bulk + mbarrier
//     complete_tx) instead of k*k per-pixel 4-byte gathers;
//   * the im2col expansion is a byte copy smem -> smem (SW128 K-major rows);
//   * CTAs are persistent over tiles: a ring of footprint stages (as many as
//     fit, so up to 23 tiles' TMA in flight), two A stages and two TMEM
//     accumulators, so the TMA of tiles i+1.., the expansion of tile i, the
//     MMAs of tile i-1 and the epilogue of tile i-2 overlap.
//
// Warp roles (18 warps): 0-7 expand A tiles, 8 issues tcgen05.mma, 9-16
// drain TMEM (recombine, bias, ReLU, store; two warps per TMEM lane
// quadrant, half the columns each), 17 issues the footprint TMA.
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "tc_bf16.cuh"

namespace ga3c {
namespace u8c {

constexpr int kBuilders = 256;
constexpr int kMmaWarp = kBuilders / 32;  // 8
constexpr int kEpilogue = 256;  // 8 warps: two per TMEM lane quadrant, half the columns each
constexpr int kTmaWarp = (kBuilders + 32 + kEpilogue) / 32;  // 17: footprint TMA producer
constexpr int kThreads = kBuilders + 32 + kEpilogue + 32;
constexpr int kFpRegion = 96 * 1024;  // footprint TMA ring: a.fp_stages stages of a.fp_bytes
constexpr int kFpMaxStages = 24;      // (the host sizes the stage to the footprint bound)
constexpr int kMaxK = 256;

struct ConvArgs {
  const uint8_t* x;   // frames, NHWC u8, frame b at x + b * bstride
  long long bstride;  // bytes between frames (multiple of 16)
  const float* w;     // [N][K] fp32 (OHWI), K = k * k * cin
  const float* bias;  // [N]
  float* out;         // [M][ldo]
  int ldo;
  int B, ih, iw, cin, k, s, oh, ow, N, K;
  int tiles;  // ceil(B * oh * ow / 128)
  int fp_bytes, fp_stages;  // footprint ring geometry (fp_bytes % 128 == 0)
};

// kind::i8 instruction descriptor: c_format S32 (2), a_format u8 (0),
// b_format s8 (1), both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_u8s8(int M, int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int BN>
struct Shape {
  static constexpr int NW = 4 * BN;                 // N-concatenated digit rows
  static constexpr int W_BYTES = NW * kMaxK;        // s8, (K/128) chunks of NW x 128 B
  static constexpr int A_BYTES = 128 * kMaxK;       // u8, (K/128) chunks of 128 x 128 B
  static constexpr int STG_BYTES = 128 * (BN + 4) * 4;  // epilogue staging
  static constexpr int SMEM = W_BYTES + 2 * A_BYTES + kFpRegion + STG_BYTES + 1024;
  static constexpr int ACC = ws::TmemCols<NW>::V;   // columns per accumulator
  static constexpr int TMEM_COLS = 2 * ACC;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Input rows y0..y1 of frame b covered by the tile's pixels in that frame.
struct Span {
  int b, y0, y1;
};

__device__ __forceinline__ void tile_spans(const ConvArgs& a, int m0, Span& s0, Span& s1, int& nimg) {
  const int P = a.oh * a.ow;
  const int M = a.B * P;
  const int m1 = min(M, m0 + 128) - 1;
  const int b0 = m0 / P, b1 = m1 / P;
  const int p0 = m0 - b0 * P, p1 = m1 - b1 * P;
  s0.b = b0;
  s0.y0 = (p0 / a.ow) * a.s;
  s0.y1 = (b1 == b0 ? p1 / a.ow : a.oh - 1) * a.s + a.k - 1;
  nimg = 1;
  if (b1 != b0) {
    s1.b = b1;
    s1.y0 = 0;
    s1.y1 = (p1 / a.ow) * a.s + a.k - 1;
    nimg = 2;
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) tc_u8conv_kernel(ConvArgs a) {
  using S = Shape<BN>;
  static_assert(4 * BN <= 256 && BN % 16 == 0, "N-concatenated tile exceeds the MMA N limit");
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t fp_full[kFpMaxStages], fp_empty[kFpMaxStages], a_full[2], a_empty[2], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_sh[BN];
  __shared__ int wmax_sh[BN];    // max |w| per output channel (float bits)
  __shared__ float scale_sh[BN];  // 2^(e_n - 38)
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sW = tc::smem_u32(smem);
  const uint32_t sA = sW + S::W_BYTES;          // 2 x A_BYTES
  const uint32_t sFp = sA + 2 * S::A_BYTES;      // a.fp_stages x a.fp_bytes
  const int NFP = a.fp_stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.y * BN;
  const int P = a.oh * a.ow;
  const int M = a.B * P;
  const int kch = a.K / 128;       // 128-byte s8/u8 row chunks
  const int rowb = a.iw * a.cin;   // bytes per input row
  const int seglen = a.k * a.cin;  // contiguous bytes per (pixel, kh)
  const int nparts = seglen / 16;
  const int ntiles = (a.tiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                     static_cast<int>(gridDim.x);

  auto issue_tma = [&](int i) {  // footprint of local tile i into stage i % NFP
    const int m0 = (static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x)) * 128;
    Span s0, s1;
    int nimg;
    tile_spans(a, m0, s0, s1, nimg);
    const uint32_t b0 = static_cast<uint32_t>((s0.y1 - s0.y0 + 1) * rowb);
    const uint32_t b0r = (b0 + 15u) & ~15u;
    const uint32_t b1 = nimg == 2 ? static_cast<uint32_t>((s1.y1 - s1.y0 + 1) * rowb) : 0u;
    const int fs = i % NFP;
    const uint32_t dst = sFp + fs * a.fp_bytes;
    mbar_expect_tx(&fp_full[fs], b0 + b1);
    bulk_g2s(dst, a.x + s0.b * a.bstride + static_cast<long long>(s0.y0) * rowb, b0, &fp_full[fs]);
    if (nimg == 2)
      bulk_g2s(dst + b0r, a.x + s1.b * a.bstride + static_cast<long long>(s1.y0) * rowb, b1, &fp_full[fs]);
  };
  pdl_trigger();
  if (tid < BN) wmax_sh[tid] = 0;
  if (warp == kMmaWarp) {
    tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
    if (lane == 0) {
      for (int i = 0; i < NFP; ++i) {
        tc::mbar_init(&fp_full[i], 1);
        tc::mbar_init(&fp_empty[i], kBuilders);
      }
      for (int i = 0; i < 2; ++i) {
        tc::mbar_init(&a_full[i], kBuilders);
        tc::mbar_init(&a_empty[i], 1);
        tc::mbar_init(&acc_full[i], 1);
        tc::mbar_init(&acc_empty[i], kEpilogue);
      }
      tc::fence_barrier_init();
    }
  }
  __syncthreads();
  pdl_wait();  // W, bias and the frames may come from the predecessor
  if (warp == kTmaWarp && lane == 0)  // the first footprints travel while the weights are prepared
    for (int j = 0; j < NFP && j < ntiles; ++j) issue_tma(j);
  // ---- weights: per-channel power-of-two grid, four exact s8 digits
  const int K4 = a.K / 4;
  const int units = BN * K4;  // 4 consecutive k of one row
  const int nthr = kThreads - 64;
  const int t = warp < kMmaWarp ? tid : tid - 32;
  const bool wprep = warp != kMmaWarp && warp != kTmaWarp;
  if (wprep) {
    for (int u = t; u < units; u += nthr) {
      const int r = u / K4;
      if (n0 + r >= a.N) continue;
      const float4 p = __ldg(reinterpret_cast<const float4*>(a.w + static_cast<std::size_t>(n0 + r) * a.K + 4 * (u - r * K4)));
      const float m = fmaxf(fmaxf(fabsf(p.x), fabsf(p.y)), fmaxf(fabsf(p.z), fabsf(p.w)));
      atomicMax(&wmax_sh[r], __float_as_int(m));
    }
  }
  __syncthreads();
  if (wprep) {
    for (int u = t; u < units; u += nthr) {
      const int r = u / K4, k0 = 4 * (u - r * K4);
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      int e = 0;
      const float mx = __int_as_float(wmax_sh[r]);
      if (n0 + r < a.N) {
        const float4 p = __ldg(reinterpret_cast<const float4*>(a.w + static_cast<std::size_t>(n0 + r) * a.K + k0));
        v[0] = p.x, v[1] = p.y, v[2] = p.z, v[3] = p.w;
        if (mx > 0.f) e = ilogbf(mx) + 1;  // 2^e > max|w|
      }
      uint32_t dig[4] = {0u, 0u, 0u, 0u};  // digit j of the 4 weights, packed bytes
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int x = mx > 0.f ? __float2int_rn(ldexpf(v[q], 30 - e)) : 0;
        // balanced base-256 digits, least significant first: d3, d2, d1, then d0 = the rest
#pragma unroll
        for (int j = 3; j >= 1; --j) {
          const int d = static_cast<int>(static_cast<int8_t>(x & 0xFF));
          x = (x - d) >> 8;
          dig[j] |= (static_cast<uint32_t>(d) & 0xFFu) << (8 * q);
        }
        dig[0] |= (static_cast<uint32_t>(x) & 0xFFu) << (8 * q);
      }
      const int c = k0 / 128, byte = k0 % 128;
      const uint32_t base = sW + c * (S::NW * 128);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = j * BN + r;
        sts32(base + tc::sw128_off(row, byte >> 4) + (byte & 15), dig[j]);
      }
    }
    if (tid < BN) {
      bias_sh[tid] = n0 + tid < a.N ? __ldg(a.bias + n0 + tid) : 0.f;
      const float mx = __int_as_float(wmax_sh[tid]);
      const int e = mx > 0.f ? ilogbf(mx) + 1 : 0;
      scale_sh[tid] = ldexpf(1.0f, e - 38);  // 2^(e-30) digit grid x 2^-8 input scale
    }
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;



  if (warp < kMmaWarp) {
    // ------------------------------------------------ A expansion
    const bool fast = a.k == 8 && nparts == 2;  // 8x8 kernels over 4 channels (GA3C conv1)
    const bool aligned16 = (a.s * a.cin) % 16 == 0 && rowb % 16 == 0;
    for (int i = 0; i < ntiles; ++i) {
      const int st = i & 1, fs = i % NFP;
      const uint32_t fp = sFp + fs * a.fp_bytes;
      const uint32_t at = sA + st * S::A_BYTES;
      tc::mbar_wait(&fp_full[fs], (i / NFP) & 1);
      if (i >= 2) tc::mbar_wait(&a_empty[st], ((i - 2) >> 1) & 1);
      const int m0 = (static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x)) * 128;
      Span s0, s1;
      int nimg;
      tile_spans(a, m0, s0, s1, nimg);
      const int b0r = (((s0.y1 - s0.y0 + 1) * rowb) + 15) & ~15;
      // two threads per pixel row r (alternate kh); a (kh, 16-byte part)
      // unit is 16 contiguous footprint bytes -> one SW128 16-byte unit
      {
        const int r = tid & 127, half = tid >> 7;
        const int m = m0 + r;
        const uint32_t drow = at + static_cast<uint32_t>(((r >> 3) << 10) | ((r & 7) << 7));
        const uint32_t key = static_cast<uint32_t>(r & 7);
        if (m < M) {
          const int b = m / P, p = m - b * P;
          const int oy = p / a.ow, ox = p - oy * a.ow;
          const bool second = nimg == 2 && b != s0.b;
          const uint32_t src0 = fp + (second ? b0r : 0) + (oy * a.s - (second ? s1.y0 : s0.y0)) * rowb +
                                ox * a.s * a.cin;
          if (fast) {
            // all loads in flight before the 8 stores; 16-byte loads when every
            // pixel's run starts 16-byte aligned (stride * cin % 16 == 0)
            uint32_t v[8][4];
            if (aligned16) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const uint32_t src = src0 + (half + 2 * (u >> 1)) * rowb + (u & 1) * 16;
                const float4 w = pipe::lds128(src);
                v[u][0] = __float_as_uint(w.x);
                v[u][1] = __float_as_uint(w.y);
                v[u][2] = __float_as_uint(w.z);
                v[u][3] = __float_as_uint(w.w);
              }
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const uint32_t src = src0 + (half + 2 * (u >> 1)) * rowb + (u & 1) * 16;
#pragma unroll
                for (int q = 0; q < 4; ++q) v[u][q] = pipe::lds32(src + 4 * q);
              }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t kpos = static_cast<uint32_t>((half + 2 * (u >> 1)) * 32 + (u & 1) * 16);
              bf::sts128u(drow + (kpos >> 7) * (128 * 128) + ((((kpos & 127) >> 4) ^ key) << 4), v[u][0], v[u][1],
                          v[u][2], v[u][3]);
            }
          } else {
            for (int kh = half; kh < a.k; kh += 2) {
              for (int part = 0; part < nparts; ++part) {
                const uint32_t src = src0 + kh * rowb + part * 16;
                const uint32_t kpos = static_cast<uint32_t>(kh * seglen + part * 16);
                bf::sts128u(drow + (kpos >> 7) * (128 * 128) + ((((kpos & 127) >> 4) ^ key) << 4),
                            pipe::lds32(src), pipe::lds32(src + 4), pipe::lds32(src + 8), pipe::lds32(src + 12));
              }
            }
          }
        } else {
          for (int kh = half; kh < a.k; kh += 2)
            for (int part = 0; part < nparts; ++part) {
              const uint32_t kpos = static_cast<uint32_t>(kh * seglen + part * 16);
              bf::sts128u(drow + (kpos >> 7) * (128 * 128) + ((((kpos & 127) >> 4) ^ key) << 4), 0u, 0u, 0u, 0u);
            }
        }
      }
      bf::mbar_arrive(&fp_empty[fs]);
      tc::fence_async_smem();
      bf::mbar_arrive(&a_full[st]);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issue
    if (lane == 0) {
      constexpr uint32_t id = idesc_u8s8(128, S::NW);
      for (int i = 0; i < ntiles; ++i) {
        const int st = i & 1;
        if (i >= 2) tc::mbar_wait(&acc_empty[st], ((i - 2) >> 1) & 1);
        tc::mbar_wait(&a_full[st], (i >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t at = sA + st * S::A_BYTES;
        const uint32_t acc = tmem + st * S::ACC;
        for (int c = 0; c < kch; ++c) {
          const uint32_t ac = at + c * (128 * 128), wc = sW + c * (S::NW * 128);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // 4 x K=32 (32 bytes) per 128-byte row
            mma_i8(acc, tc::sdesc_sw128(ac + kk * 32, 16, 1024), tc::sdesc_sw128(wc + kk * 32, 16, 1024), id,
                   (c | kk) != 0);
        }
        tc::mma_commit(&a_empty[st]);
        tc::mma_commit(&acc_full[st]);
      }
    }
    __syncwarp();
  } else if (warp == kTmaWarp) {
    // ------------------------------------------------ footprint TMA producer
    if (lane == 0)
      for (int j = NFP; j < ntiles; ++j) {
        // stage j % NFP last held tile j - NFP: every builder must be done with it
        tc::mbar_wait(&fp_empty[j % NFP], ((j - NFP) / NFP) & 1);
        issue_tma(j);
      }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue (8 warps: lane quadrant x column half)
    const int quad = warp & 3;
    const int ew = warp - (kMmaWarp + 1);  // 0..7
    constexpr int HB = BN / 2;              // columns per warp
    const int cb = (ew >> 2) * HB;
    constexpr int PR = BN + 4;  // staging pitch (floats)
    float* stg = reinterpret_cast<float*>(smem + S::W_BYTES + 2 * S::A_BYTES + kFpRegion) +
                 quad * 32 * PR;
    for (int i = 0; i < ntiles; ++i) {
      const int st = i & 1;
      tc::mbar_wait(&acc_full[st], (i >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t trow = tmem + st * S::ACC + (static_cast<uint32_t>(quad * 32) << 16) + cb;
#pragma unroll
      for (int c0 = 0; c0 < HB; c0 += 8) {
        float d0[8], d1[8], d2[8], d3[8];
        tc::tmem_ld8(trow + c0, d0);
        tc::tmem_ld8(trow + BN + c0, d1);
        tc::tmem_ld8(trow + 2 * BN + c0, d2);
        tc::tmem_ld8(trow + 3 * BN + c0, d3);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; j += 4) {
          float o[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            // exact s32 digit sums, combined smallest first in fp32
            const int c = cb + c0 + j + u;
            const float f = ((static_cast<float>(__float_as_int(d3[j + u])) +
                              static_cast<float>(__float_as_int(d2[j + u])) * 256.0f) +
                             static_cast<float>(__float_as_int(d1[j + u])) * 65536.0f) +
                            static_cast<float>(__float_as_int(d0[j + u])) * 16777216.0f;
            o[u] = bf::relu(fmaf(f, scale_sh[c], bias_sh[c]));
          }
          bf::sts128u(tc::smem_u32(stg + lane * PR + cb + c0 + j), __float_as_uint(o[0]), __float_as_uint(o[1]),
                      __float_as_uint(o[2]), __float_as_uint(o[3]));
        }
      }
      tc::tc_fence_before();
      bf::mbar_arrive(&acc_empty[st]);
      __syncwarp();
      // the quad's 32 rows are 32 consecutive pixels: this warp's column half, float4 rows
      const int mq = (static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x)) * 128 + quad * 32;
      constexpr int V4 = HB / 4;
      for (int e = lane; e < 32 * V4; e += 32) {
        const int rr = e / V4, q4 = e - rr * V4;
        const int m = mq + rr;
        const int col = cb + 4 * q4;
        if (m < M && n0 + col < a.N)
          *reinterpret_cast<float4*>(a.out + static_cast<std::size_t>(m) * a.ldo + n0 + col) =
              pipe::lds128(tc::smem_u32(stg + rr * PR + col));
      }
      __syncwarp();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace u8c
}  // namespace ga3c
