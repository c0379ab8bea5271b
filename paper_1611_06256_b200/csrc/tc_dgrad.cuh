// tc_dgrad.cuh -- conv input gradient on the tensor cores (kind::tf32, 3xTF32).
//
// The input gradient of a VALID conv with kernel k and stride s
// (nnet.cpp:273-277 restated for conv: dx = W^T g, gated by the ReLU of the
// layer below, nnet.cpp:268-271) is a transposed conv.  Split the input
// pixels into s*s stride phases (ih = s*a + p, iw = s*b + q): within a phase
// only the taps kh = p + s*j, kw = q + s*l (j, l < T = k/s) reach the pixel,
// from output pixel (a - j, b - l).  So each phase is a dense implicit GEMM
//
//   dX_pq[(n,a,b)][ci] = sum_{j,l,co} dY[n, a-j, b-l, co] * W[co, p+s*j, q+s*l, ci]
//
// with M = B * ceil((IH-p)/s) * ceil((IW-q)/s), N = Cin, K = T*T*Cout, no
// wasted products, and zero-filled rows where a-j or b-l falls outside the
// output map.  The phases are grid.y; the ReLU gate of the layer below is
// fused into the store.
//
// Structure is tc_kk_ws_kernel's (tc_ws.cuh): 8 producer warps gather 32-wide
// k chunks with cp.async (dY rows: 16-byte vectors, one tap per chunk since
// Cout % 32 == 0; W: 4-byte transposing gathers into the K-major tile), derive
// the tf32 lo halves in place and signal ready[]; one MMA warp issues
//   A_hi x [W_hi ; W_lo]  (N = 2*BN, N-concatenated)  and  A_lo x W_hi (N = BN)
// per 8-wide k step; the epilogue adds the two TMEM column ranges.
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "tc_pipe.cuh"
#include "tc_ws.cuh"

namespace ga3c {
namespace dg {

struct DgradArgs {
  const float* dy;    // [B][OH][OW][cout]
  const float* w;     // [cout][k][k][cin]
  const float* gate;  // [B][IH][IW][cin] post-activation of the layer below
  float* dx;          // [B][IH][IW][cin]
  int B, IH, IW, cin, OH, OW, cout, k, s, T;
};

template <int BN, int CAP>
struct DgShape {
  static constexpr int A_HI = 128 * 128;     // 128 rows x 32 fp32
  static constexpr int A_BYTES = 2 * A_HI;   // hi + lo
  static constexpr int B_HI = BN * 128;
  static constexpr int B_BYTES = 2 * B_HI;   // hi rows [0,BN) then lo rows [BN,2BN)
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NS = pipe::ring_depth(CAP, STAGE);
  static constexpr int SMEM = NS * STAGE + 1024;
  static constexpr int TMEM_COLS = ws::TmemCols<2 * BN>::V;
  static constexpr int AV = 128 * 8 / ws::kProducers;  // 16-byte A vectors per producer thread
  static constexpr int BE = BN * 32;                   // B elements per chunk
  static constexpr int BPER = (BE + ws::kProducers - 1) / ws::kProducers;
};

// Register cap: two 288-thread CTAs per SM (ring caps 1-2) need <= 96
// registers per thread -- each SM sub-partition holds 5 of the 18 warps in
// 16K registers.  Uncapped (104) the occupancy limit was one CTA per SM
// (ncu launch__occupancy_limit_registers = 1) and large s1's conv2 dgrad
// took 112 us instead of 71.
template <int BN, int CAP>
__global__ void __launch_bounds__(ws::kThreads) __maxnreg__((CAP == 1 || CAP == 2) && BN <= 64 ? 96 : 255)
    tc_dgrad_kernel(DgradArgs a) {
  using S = DgShape<BN, CAP>;
  static_assert(BN % 16 == 0 && 2 * BN <= 256, "N-concatenated tile exceeds the MMA N limit");
  constexpr int kP = ws::kProducers;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t ready[pipe::kMaxStages], done[pipe::kMaxStages], acc_bar;
  __shared__ uint32_t tmem_base_sh;
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sbase = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int phase = blockIdx.y;
  const int p = phase / a.s, q = phase - (phase / a.s) * a.s;
  const int Ap = (a.IH - p + a.s - 1) / a.s, Bq = (a.IW - q + a.s - 1) / a.s;
  const int per_img = Ap * Bq;
  const int M = a.B * per_img;
  const int m0 = blockIdx.x * 128;
  if (m0 >= M || Ap <= 0 || Bq <= 0) return;  // this phase has fewer tiles
  const int n0 = blockIdx.z * BN;
  const int nchunks = a.T * a.T * a.cout / 32;

  // producer rows: thread owns A vectors idx = tid + kP*j -> row idx>>3, 16-byte v = idx&7
  int rbase[S::AV], ra[S::AV], rb[S::AV];
  uint32_t asoff[S::AV];
  auto issue = [&](int c, uint32_t st) {
    const int k0 = 32 * c;
    const int t = k0 / a.cout, co0 = k0 - t * a.cout;
    const int tj = t / a.T, tl = t - tj * a.T;
    const int shift = (tj * a.OW + tl) * a.cout - co0;
#pragma unroll
    for (int j = 0; j < S::AV; ++j) {
      const int v = (tid + kP * j) & 7;
      const bool ok = rbase[j] >= 0 && static_cast<unsigned>(ra[j] - tj) < static_cast<unsigned>(a.OH) &&
                      static_cast<unsigned>(rb[j] - tl) < static_cast<unsigned>(a.OW);
      pipe::cp16(st + asoff[j], a.dy + (ok ? rbase[j] - shift + 4 * v : 0), ok);
    }
    // W[co0+kk][p + s*tj][q + s*tl][n0 + ci] -> B tile row ci, k column kk
    const int kh = p + a.s * tj, kw = q + a.s * tl;
    const float* wsrc = a.w + static_cast<std::size_t>(co0) * a.k * a.k * a.cin + (kh * a.k + kw) * a.cin + n0;
    const int costride = a.k * a.k * a.cin;
    const uint32_t stb = st + S::A_BYTES;
#pragma unroll
    for (int j = 0; j < S::BPER; ++j) {
      const int e = tid + kP * j;
      if (e >= S::BE) break;
      const int kk = e / BN, ci = e - (e / BN) * BN;
      const bool ok = n0 + ci < a.cin;
      pipe::cp4(stb + tc::sw128_off(ci, kk >> 2) + 4 * (kk & 3), wsrc + (ok ? kk * costride + ci : 0), ok);
    }
  };

  pdl_trigger();
  if (warp < ws::kMmaWarp) {
#pragma unroll
    for (int j = 0; j < S::AV; ++j) {
      const int idx = tid + kP * j;
      const int r = idx >> 3, v = idx & 7;
      const int g = m0 + r;
      asoff[j] = tc::sw128_off(r, v);
      if (g < M) {
        const int n = g / per_img, rem = g - n * per_img;
        ra[j] = rem / Bq;
        rb[j] = rem - ra[j] * Bq;
        rbase[j] = ((n * a.OH + ra[j]) * a.OW + rb[j]) * a.cout;
      } else {
        ra[j] = rb[j] = -1 << 20;
        rbase[j] = -1;
      }
    }
    pdl_wait();
#pragma unroll
    for (int c = 0; c < S::NS - 1; ++c) {
      if (c < nchunks) issue(c, sbase + c * S::STAGE);
      pipe::commit();
    }
  } else {
    tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S::NS; ++s) {
        tc::mbar_init(&ready[s], kP);
        tc::mbar_init(&done[s], 1);
      }
      tc::mbar_init(&acc_bar, 1);
      tc::fence_barrier_init();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == ws::kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t id_cat = tc::idesc_tf32(128, 2 * BN, false, false);
      constexpr uint32_t id_one = tc::idesc_tf32(128, BN, false, false);
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % S::NS;
        tc::mbar_wait(&ready[s], (i / S::NS) & 1);
        tc::tc_fence_after();
        const uint32_t st = sbase + s * S::STAGE;
        const uint32_t ah = st, al = st + S::A_HI, bh = st + S::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t dah = tc::sdesc_sw128(ah + kk * 32, 16, 1024);
          const uint64_t dbh = tc::sdesc_sw128(bh + kk * 32, 16, 1024);
          tc::mma_tf32(tmem, dah, dbh, id_cat, (i | kk) != 0);
          tc::mma_tf32(tmem, tc::sdesc_sw128(al + kk * 32, 16, 1024), dbh, id_one, 1);
        }
        tc::mma_commit(&done[s]);
      }
      tc::mma_commit(&acc_bar);
    }
    __syncwarp();
  } else {
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % S::NS;
      const uint32_t st = sbase + s * S::STAGE;
      pipe::wait_group<S::NS - 2>();
      // lo halves in place: A (this thread's own vectors), B (hi rows -> lo rows)
#pragma unroll
      for (int j = 0; j < S::AV; ++j)
        detail::sts128(st + S::A_HI + asoff[j], pipe::lo4(pipe::lds128(st + asoff[j])));
      // B: hi rows were written by other threads' 4-byte copies
      asm volatile("bar.sync 1, %0;" ::"n"(kP) : "memory");
      const uint32_t stb = st + S::A_BYTES;
      for (int e = tid; e < BN * 8; e += kP) {
        const uint32_t off = tc::sw128_off(e >> 3, e & 7);
        detail::sts128(stb + S::B_HI + off, pipe::lo4(pipe::lds128(stb + off)));
      }
      tc::fence_async_smem();
      ws::mbar_arrive(&ready[s]);
      const int nc = i + S::NS - 1;
      if (nc < nchunks) {
        const int ps = nc % S::NS;
        if (i >= 1) tc::mbar_wait(&done[ps], ((i - 1) / S::NS) & 1);
        issue(nc, sbase + ps * S::STAGE);
      }
      pipe::commit();
    }
    // ---- epilogue: row r (TMEM lane) = pixel (n, s*a+p, s*b+q); BN channels
    if (nchunks > 0) tc::mbar_wait(&acc_bar, 0);
    tc::tc_fence_after();
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int cbeg = (warp >> 2) * HALF;
    const int g = m0 + r;
    std::size_t off = 0;
    if (g < M) {
      const int n = g / per_img, rem = g - n * per_img;
      const int aa = rem / Bq, bb = rem - aa * Bq;
      off = ((static_cast<std::size_t>(n) * a.IH + a.s * aa + p) * a.IW + a.s * bb + q) * a.cin + n0;
    }
    if (cbeg < BN) {
#pragma unroll 1
      for (int c = 0; c < HALF; c += 16) {
        const int c0 = cbeg + c;
        float v[16], w[16];
        const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        tc::tmem_ld16(trow + c0, v);
        tc::tmem_ld16(trow + BN + c0, w);
        tc::tmem_ld_wait();
        if (g < M) {
          if (n0 + c0 + 16 <= a.cin) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const float4 gt = __ldg(reinterpret_cast<const float4*>(a.gate + off + c0 + j));
              float4 o;
              o.x = gt.x <= 0.f ? 0.f : v[j] + w[j];
              o.y = gt.y <= 0.f ? 0.f : v[j + 1] + w[j + 1];
              o.z = gt.z <= 0.f ? 0.f : v[j + 2] + w[j + 2];
              o.w = gt.w <= 0.f ? 0.f : v[j + 3] + w[j + 3];
              *reinterpret_cast<float4*>(a.dx + off + c0 + j) = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + c0 + j < a.cin) a.dx[off + c0 + j] = a.gate[off + c0 + j] <= 0.f ? 0.f : v[j] + w[j];
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == ws::kMmaWarp) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace dg
}  // namespace ga3c
