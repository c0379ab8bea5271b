// tc_wgrad_band.cuh -- weight gradient of the u8 first conv layer
// (nnet.cpp:58-73 summed over the batch) when one window row is k * Cin = 32
// contiguous bytes (GA3C's conv1: 8x8 over the 4-frame stack, both nets):
//
//   dW[co][kk] = sum_p X(p, kk) dY(p, co)        db[co] = sum_p dY(p, co)
//
// The im2col path (tc_mn_ws_kernel<uint8_t>) fetches every 32-byte window
// row of every output pixel from L2 with 4-byte cp.async: each input byte
// k^2/s^2 times (4x for DNN A), ~1000 LSU ops per 32-pixel chunk, one global
// round trip per chunk on the CTA's critical path.  Here CTA (j, b) owns the
// 32-pixel chunks [j*cpc, (j+1)*cpc) of image b.  One thread bulk-copies the
// input rows those pixels' windows cover (contiguous in NHWC) and the
// pixels' dY rows into shared memory -- two cp.async.bulk on one mbarrier;
// then the 8 producer warps build each chunk's MN-major operands shared ->
// shared (u8 widened exactly to fp32 for X; dY as tf32 hi and lo halves, as
// in tc_mn_ws_kernel) into a 2-stage ring, and the MMA warp issues MT x 4
// tcgen05.mma (kind::tf32, M = 128 kk, N = 2 x 32 co hi|lo, K = 8 pixels)
// per chunk into TMEM.  The partials [split][cout][Kw] (+ bias column) go to
// the same fixed-order split-K reduction as the im2col path (split = b * cpi
// + j), so the result is deterministic for a given plan.
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "tc_pipe.cuh"
#include "tc_wgrad.cuh"

namespace ga3c {
namespace wb {

struct BandArgs {
  const uint8_t* x;  // images, bstride bytes apart, NHWC u8
  long long bstride;
  int iw, cin, k, stride, ow, P;  // P = output pixels per image
  const float* D;                 // [B * P][ldd] output gradient (ReLU-gated)
  int ldd, cout, Kw;              // Kw = k * 32
  int cpi, cpc;                   // CTAs per image, 32-pixel chunks per CTA
  int xband, dband;               // shared bytes reserved for input rows / dY rows
  int splits;                     // cpi * B
  float* part;                    // [splits][cout][Kw], then [splits][cout] bias
  GradMap gm;
  int direct;  // splits == 1: store into dtheta
};

constexpr int kProducers = 256;  // 8 producer warps
constexpr int kThreads = kProducers + 32;
constexpr int kMmaWarp = kProducers / 32;
constexpr int BN = 32;                 // output channels per MMA (cout <= 32, zero padded)
constexpr int NS = 2;                  // operand ring depth
constexpr int X_SBO = 4 * 512;         // 4 MN atoms of 32 kk per 4-pixel k group
constexpr int X_BYTES = 32 * 128 * 4;  // one 128-kk tile of a 32-pixel chunk
constexpr int D_SBO = 2 * 512;         // hi atom + lo atom per k group
constexpr int D_BYTES = 32 * 2 * BN * 4;
constexpr int PT = 128 + 4;            // epilogue staging row pitch (floats)

template <int MT>
struct Shape {
  static constexpr int STAGE = MT * X_BYTES + D_BYTES;
  static constexpr int RING = NS * STAGE;
  static constexpr int TMEM_COLS = MT * 2 * BN <= 64 ? 64 : 128;
  static_assert(BN * PT * 4 <= RING, "epilogue staging reuses the ring");
};

__host__ __device__ constexpr int smem_bytes(int mt, int xband, int dband) {
  return (mt == 1 ? Shape<1>::RING : Shape<2>::RING) + xband + dband + 1024;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

template <int MT>
__global__ void __launch_bounds__(kThreads, 1) tc_wgrad_band_kernel(BandArgs a) {
  using S = Shape<MT>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t ready[NS], done[NS], band_bar, acc_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_red[32][BN + 1];
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sbase = tc::smem_u32(smem);
  const uint32_t xb = sbase + S::RING;  // input rows y0 .. y1-1 of image b
  const uint32_t db = xb + a.xband;     // dY rows of pixels p0 .. p1-1
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = blockIdx.x, b = blockIdx.y;
  const int split = b * a.cpi + j;
  const int c0 = j * a.cpc;
  const int c1 = min((a.P + 31) / 32, c0 + a.cpc);
  const int nchunks = max(0, c1 - c0);
  const int p0 = 32 * c0;
  const int p1 = min(a.P, 32 * c1);
  const int rowb = a.iw * a.cin;
  const int y0 = nchunks > 0 ? (p0 / a.ow) * a.stride : 0;
  const int y1 = nchunks > 0 ? ((p1 - 1) / a.ow) * a.stride + a.k : 0;

  pdl_trigger();
  if (warp == kMmaWarp) {
    tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        tc::mbar_init(&ready[s], kProducers);
        tc::mbar_init(&done[s], 1);
      }
      tc::mbar_init(&band_bar, 1);
      tc::mbar_init(&acc_bar, 1);
      tc::fence_barrier_init();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  pdl_wait();  // dY comes from the previous kernel; the partials may still be read by the last reduction
  if (tid == 0 && nchunks > 0) {
    const uint32_t xbytes = static_cast<uint32_t>((y1 - y0) * rowb);
    const uint32_t dbytes = static_cast<uint32_t>((p1 - p0) * a.ldd * 4);
    tc::mbar_expect_tx(&band_bar, xbytes + dbytes);
    tc::bulk_g2s(xb, a.x + b * a.bstride + static_cast<long long>(y0) * rowb, xbytes, &band_bar);
    tc::bulk_g2s(db, a.D + (static_cast<std::size_t>(b) * a.P + p0) * a.ldd, dbytes, &band_bar);
  }

  if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t id = tc::idesc_tf32(128, 2 * BN, true, true);
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % NS;
        tc::mbar_wait(&ready[s], (i / NS) & 1);
        tc::tc_fence_after();
        const uint32_t st = sbase + s * S::STAGE;
        const uint32_t dt = st + MT * X_BYTES;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {  // 8 pixels = two 4-row k groups per MMA
            const uint64_t da = tc::sdesc(st + mt * X_BYTES + 2 * h * X_SBO, 512, X_SBO, 1);
            const uint64_t dd = tc::sdesc(dt + 2 * h * D_SBO, 512, D_SBO, 1);
            tc::mma_tf32(tmem + mt * 2 * BN, da, dd, id, (i | h) != 0);
          }
        }
        tc::mma_commit(&done[s]);
      }
      tc::mma_commit(&acc_bar);
    }
  } else {
    // thread -> (pixel row xp of the chunk, 16-byte vector xv): X atoms of
    // that pixel's window rows, dY channels 4xv .. 4xv+3
    const int xp = tid >> 3, xv = tid & 7;
    uint32_t xoff[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) xoff[g] = detail::mn_off(xp, g, xv, X_SBO);
    const uint32_t doff_hi = detail::mn_off(xp, 0, xv, D_SBO), doff_lo = detail::mn_off(xp, 1, xv, D_SBO);
    float4 bs = make_float4(0.f, 0.f, 0.f, 0.f);
    // this thread's pixel (oy, ox), advanced by 32 pixels per chunk without a division
    int oy = (p0 + xp) / a.ow, ox = (p0 + xp) - ((p0 + xp) / a.ow) * a.ow;
    const int dy = 32 / a.ow, dx = 32 - (32 / a.ow) * a.ow;
    if (nchunks > 0) tc::mbar_wait(&band_bar, 0);
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % NS;
      if (i >= NS) tc::mbar_wait(&done[s], ((i / NS) - 1) & 1);
      const uint32_t st = sbase + s * S::STAGE;
      const int p = p0 + 32 * i + xp;
      const bool pv = p < p1;
      // branch-free: every load is issued (invalid ones from the band's
      // first word) before any is used, then invalid lanes select zero
      const uint32_t src =
          pv ? xb + static_cast<uint32_t>((oy * a.stride - y0) * rowb + ox * a.stride * a.cin + 4 * xv) : xb;
      uint32_t w[4 * MT];
#pragma unroll
      for (int q = 0; q < 4 * MT; ++q) w[q] = pipe::lds32(src + (q < a.k ? q : 0) * rowb);
      const bool dv = pv && 4 * xv < a.cout;
      float4 d = pipe::lds128(dv ? db + static_cast<uint32_t>(((p - p0) * a.ldd + 4 * xv) * 4) : db);
      if (!dv) d = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 4 * MT; ++q) {
        float4 f = pipe::widen_u8(w[q]);
        if (!pv || q >= a.k) f = make_float4(0.f, 0.f, 0.f, 0.f);
        detail::sts128(st + (q >> 2) * X_BYTES + xoff[q & 3], f);
      }
      bs.x += d.x;
      bs.y += d.y;
      bs.z += d.z;
      bs.w += d.w;
      const uint32_t dt = st + MT * X_BYTES;
      detail::sts128(dt + doff_hi, d);
      detail::sts128(dt + doff_lo, pipe::lo4(d));
      tc::fence_async_smem();
      mbar_arrive(&ready[s]);
      oy += dy;
      ox += dx;
      if (ox >= a.ow) {
        ox -= a.ow;
        ++oy;
      }
    }
    // ---- epilogue: C'[kk][co] staged transposed as [co][kk], whole 128-kk
    // rows stored with float4s; bias = fixed-order sum over the 32 pixel rows
    bias_red[xp][4 * xv + 0] = bs.x;
    bias_red[xp][4 * xv + 1] = bs.y;
    bias_red[xp][4 * xv + 2] = bs.z;
    bias_red[xp][4 * xv + 3] = bs.w;
    if (nchunks > 0) tc::mbar_wait(&acc_bar, 0);
    tc::tc_fence_after();
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    constexpr int HALF = BN / 2;
    const int cbeg = (warp >> 2) * HALF;
    float* stg = reinterpret_cast<float*>(smem);  // the ring: every MMA has completed
    const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
#pragma unroll 1
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll 1
      for (int c = 0; c < HALF; c += 16) {
        const int cc = cbeg + c;
        float v[16];
        if (nchunks > 0) {
          float w[16];
          tc::tmem_ld16(trow + mt * 2 * BN + cc, v);
          tc::tmem_ld16(trow + mt * 2 * BN + BN + cc, w);
          tc::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] += w[q];
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) stg[(cc + q) * PT + r] = v[q];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
      const int kk0 = 128 * mt;
      const bool lane_ok = kk0 + 4 * lane < a.Kw;
#pragma unroll
      for (int q = 0; q < BN / 8; ++q) {
        const int co = warp + 8 * q;
        if (co >= a.cout) break;
        const float4 x = *reinterpret_cast<const float4*>(stg + co * PT + 4 * lane);
        if (a.direct) {
          bool bad = false;
          if (lane_ok) {
            *reinterpret_cast<float4*>(a.gm.dtheta + a.gm.w0 + static_cast<std::size_t>(co) * a.Kw + kk0 +
                                       4 * lane) = x;
            bad = !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
          }
          if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.gm.flag, 1);
        } else if (lane_ok) {
          *reinterpret_cast<float4*>(a.part + (static_cast<std::size_t>(split) * a.cout + co) * a.Kw + kk0 +
                                     4 * lane) = x;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");  // staging reused by the next tile
    }
    if (tid < a.cout) {
      float t = 0.f;
      for (int q = 0; q < 32; ++q) t += bias_red[q][tid];
      if (a.direct)
        a.gm.store(tid, a.Kw, t);
      else
        a.part[static_cast<std::size_t>(a.splits) * a.cout * a.Kw + static_cast<std::size_t>(split) * a.cout + tid] =
            t;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace wb
}  // namespace ga3c
