// tc_ws.cuh -- warp-specialized tcgen05 GEMMs (kind::tf32, 3xTF32) used by
// the GA3C trunk: 8 producer warps stream operand chunks with cp.async into
// an S-stage shared-memory ring and derive the tf32 "lo" halves in place; a
// ninth warp only issues tcgen05.mma and commits completion, so MMA issue
// never sits on the producers' critical path (ready[]/done[] mbarriers).
//
// tcgen05.mma has a ~48-cycle issue floor per instruction for N <= 64 (M=128,
// K=8; measured on B200 by tools/mma_rate.cu), so the 3xTF32 product
//   A_hi*B_hi + A_hi*B_lo + A_lo*B_hi
// is issued as two instructions per k-step: A_hi x [B_hi ; B_lo] with
// N = 2*BN (the two halves land in adjacent TMEM column ranges) and
// A_lo x B_hi with N = BN accumulated onto the first range; the epilogue adds
// the two ranges.  u8 frames are exact in tf32 and skip A_lo.
//
//   tc_kk_ws_kernel : C[m][n] = sum_k A(m,k) B(n,k), K-major operands
//                     (conv / FC forward; Seg + TcEpiArgs contract)
//   tc_mn_ws_kernel : C'[kk][co] = sum_m X(m,kk) D(m,co), MN-major operands
//                     (weight gradients, transposed FC input gradient;
//                     WgradArgs contract)
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "tc_pipe.cuh"

namespace ga3c {
namespace ws {

using pipe::commit;
using pipe::cp16;
using pipe::cp4;
using pipe::lds128;
using pipe::lds32;
using pipe::lo4;
using pipe::wait_group;
using pipe::widen_u8;

constexpr int kProducers = 256;            // 8 producer warps
constexpr int kThreads = kProducers + 32;  // + the MMA warp
constexpr int kMmaWarp = kProducers / 32;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

template <int COLS>
struct TmemCols {
  static constexpr int V = COLS <= 32 ? 32 : (COLS <= 64 ? 64 : (COLS <= 128 ? 128 : (COLS <= 256 ? 256 : 512)));
};

// =========================================================== K-major GEMM
// CAP (pipe::ring_depth): 1 = at most ~100 KB of ring so two CTAs share an SM (multi-wave
// grids: the second CTA's loads and MMAs cover the first one's epilogue).
template <typename TA, typename TB, int BN, int CAP = 0>
struct KKShape {
  using TileA = pipe::KTile<TA, 128>;
  using TileB = pipe::KTile<TB, BN>;  // f32: hi rows [0,BN) then lo rows [BN,2BN) -- one 2BN-row tile
  static constexpr bool A_LO = sizeof(TA) == 4;
  static constexpr bool B_LO = sizeof(TB) == 4;
  static constexpr int STAGE = TileA::BYTES + TileB::BYTES;
  static constexpr int NS_DEEP = pipe::stages_for(STAGE);
  static constexpr int NS = pipe::ring_depth(CAP, STAGE);
  static_assert(NS_DEEP >= 2, "tile too large for a 2-stage pipeline");
  static constexpr int SMEM = NS * STAGE + 1024;
  static constexpr int ACC_COLS = B_LO ? 2 * BN : BN;
  static constexpr int TMEM_COLS = TmemCols<ACC_COLS>::V;
};

// TMA (conv forward, fp32 operands): one producer thread loads each stage's
// hi tiles with an im2col tensor copy (A) and a tiled copy (B) that complete
// on full[s]; the producer warps then only compute the lo parts.
template <typename TA, typename TB, int BN, int MODE, int CAP = 0, bool TMA = false>
__global__ void __launch_bounds__(kThreads, 1)
tc_kk_ws_kernel(Seg A, Seg B, int M, int N, int K, int kc, TcEpiArgs epi, const __grid_constant__ TmaConv tm) {
  using S = KKShape<TA, TB, BN, CAP>;
  static_assert(!S::B_LO || 2 * BN <= 256, "N-concatenated tile exceeds the MMA N limit");
  static_assert(!TMA || (sizeof(TA) == 4 && sizeof(TB) == 4 && MODE == TC_EPI_BIAS_RELU), "TMA: fp32 conv forward");
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t ready[pipe::kMaxStages], done[pipe::kMaxStages], full[pipe::kMaxStages], acc_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_sh[BN];
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sbase = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.z * BN;
  const int split = blockIdx.y;
  const int kb = split * kc;
  const int ke = min(K, kb + kc);
  const int nchunks = (ke - kb + 31) / 32;
  // BIAS_RELU with grid.y > 1: split-K over a (1, grid.y, 1) cluster
  const bool csplit = MODE == TC_EPI_BIAS_RELU && gridDim.y > 1;

  TRACE(0);
  typename S::TileA ta;
  typename S::TileB tb;
  // TMA: the first output pixel's window corner (b, h, w) in the input
  int t_w = 0, t_h = 0, t_n = 0;
  auto tma_issue = [&](int c, uint32_t st, uint64_t* bar) {
    const int k0 = kb + 32 * c;
    const int tap = k0 / tm.cin, ci0 = k0 - tap * tm.cin;
    const int ky = tap / tm.k, kx = tap - ky * tm.k;
    tc::mbar_expect_tx(bar, S::TileA::HI_BYTES + S::TileB::HI_BYTES);
    tc::tma_im2col_4d(st, &tm.a, ci0, t_w, t_h, t_n, static_cast<uint16_t>(kx), static_cast<uint16_t>(ky), bar);
    tc::tma_tile_2d(st + S::TileA::BYTES, &tm.b, k0, n0, bar);
  };
  if constexpr (TMA) {
    const int pp = m0 % A.P, oy = pp / A.ow;
    t_n = m0 / A.P;
    t_h = oy * tm.stride;
    t_w = (pp - oy * A.ow) * tm.stride;
  }
  pdl_trigger();
  if (warp < kMmaWarp) {
    ta.init(A, m0, tid);
    tb.init(B, n0, tid);
    if constexpr (TMA) {
      pdl_wait();  // the epilogue's global accesses, and the loads below, follow the predecessor
      if (tid == 0) {
        tc::tma_prefetch_desc(&tm.a);
        tc::tma_prefetch_desc(&tm.b);
#pragma unroll
        for (int s = 0; s < S::NS; ++s) tc::mbar_init(&full[s], 1);
        tc::fence_barrier_init();
      }
    } else {
      pdl_wait();  // everything below reads the predecessor's outputs
#pragma unroll
      for (int c = 0; c < S::NS - 1; ++c) {
        if (c < nchunks) {
          const uint32_t st = sbase + c * S::STAGE;
          ta.issue(A, A.chunkoff(kb + 32 * c), st, tid);
          tb.issue(B, B.chunkoff(kb + 32 * c), st + S::TileA::BYTES, tid);
        }
        commit();
      }
    }
  } else {
    tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S::NS; ++s) {
        tc::mbar_init(&ready[s], kProducers);
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
  if constexpr (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < S::NS - 1; ++c)
        if (c < nchunks) tma_issue(c, sbase + c * S::STAGE, &full[c]);
    }
  }
  TRACE(1);

  if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t id_cat = tc::idesc_tf32(128, S::B_LO ? 2 * BN : BN, false, false);
      constexpr uint32_t id_one = tc::idesc_tf32(128, BN, false, false);
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % S::NS;
        tc::mbar_wait(&ready[s], (i / S::NS) & 1);
#ifdef GA3C_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_trace[8 + 2 * i] = t_;
        }
#endif
        tc::tc_fence_after();
        const uint32_t st = sbase + s * S::STAGE;
        const uint32_t stb = st + S::TileA::BYTES;
        const uint32_t ah = ta.hi(st), al = ta.lo(st), bh = tb.hi(stb);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t dah = tc::sdesc_sw128(ah + kk * 32, 16, 1024);
          const uint64_t dbh = tc::sdesc_sw128(bh + kk * 32, 16, 1024);
          tc::mma_tf32(tmem, dah, dbh, id_cat, (i | kk) != 0);
          if constexpr (S::A_LO)
            tc::mma_tf32(tmem, tc::sdesc_sw128(al + kk * 32, 16, 1024), dbh, id_one, 1);
        }
        tc::mma_commit(&done[s]);
#ifdef GA3C_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_trace[9 + 2 * i] = t_;
        }
#endif
      }
      tc::mma_commit(&acc_bar);
    }
  } else {
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % S::NS;
      const uint32_t st = sbase + s * S::STAGE;
      if constexpr (TMA)
        tc::mbar_wait(&full[s], (i / S::NS) & 1);
      else
        wait_group<S::NS - 2>();
      TRACE(64 + 4 * i);
      ta.convert(st, tid);
      tb.convert(st + S::TileA::BYTES, tid);
      tc::fence_async_smem();
      mbar_arrive(&ready[s]);
      const int nc = i + S::NS - 1;
      if (nc < nchunks) {
        const int ps = nc % S::NS;
        const uint32_t pst = sbase + ps * S::STAGE;
        if constexpr (TMA) {
          if (tid == 0) {
            if (i >= 1) tc::mbar_wait(&done[ps], ((i - 1) / S::NS) & 1);
            tma_issue(nc, pst, &full[ps]);
          }
        } else {
          if (i >= 1) tc::mbar_wait(&done[ps], ((i - 1) / S::NS) & 1);
          ta.issue(A, A.chunkoff(kb + 32 * nc), pst, tid);
          tb.issue(B, B.chunkoff(kb + 32 * nc), pst + S::TileA::BYTES, tid);
        }
      }
      if constexpr (!TMA) commit();
    }
    // ---- epilogue (producer warps): C = acc[0:BN) (+ acc[BN:2BN) for B_lo),
    // staged through the (now idle) pipeline smem so global stores are
    // 16-byte, fully coalesced rows.
    TRACE(5);
    if constexpr (MODE == TC_EPI_BIAS_RELU) {
      // bias for this N tile, fetched while the last MMAs drain
      if (tid < BN) bias_sh[tid] = n0 + tid < N ? __ldg(epi.bias + n0 + tid) : 0.f;
      asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
    }
    if (nchunks > 0) tc::mbar_wait(&acc_bar, 0);
    tc::tc_fence_after();
    TRACE(2);
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // accumulator row (TMEM lane)
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int cbeg = (warp >> 2) * HALF;
    float* stg = reinterpret_cast<float*>(smem);
    constexpr int PR = BN + 4;   // BIAS_RELU staging [128][BN] (pitch PR)
    constexpr int PT = 128 + 4;  // PART_T staging   [BN][128] (pitch PT)
    if (cbeg < BN) {
#pragma unroll 1
      for (int c = 0; c < HALF; c += 16) {
        const int c0 = cbeg + c;
        float v[16];
        const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        tc::tmem_ld16(trow + c0, v);
        if constexpr (S::B_LO) {
          float w[16];
          tc::tmem_ld16(trow + BN + c0, w);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += w[j];
        } else {
          tc::tmem_ld_wait();
        }
        if (MODE == TC_EPI_BIAS_RELU && csplit) {
          // split-K partial: raw sums, reduced across the cluster below
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(stg + r * PR + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else if constexpr (MODE == TC_EPI_BIAS_RELU) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 q;
            q.x = v[j] + bias_sh[c0 + j];
            q.y = v[j + 1] + bias_sh[c0 + j + 1];
            q.z = v[j + 2] + bias_sh[c0 + j + 2];
            q.w = v[j + 3] + bias_sh[c0 + j + 3];
            q.x = q.x < 0.f ? 0.f : q.x;
            q.y = q.y < 0.f ? 0.f : q.y;
            q.z = q.z < 0.f ? 0.f : q.z;
            q.w = q.w < 0.f ? 0.f : q.w;
            *reinterpret_cast<float4*>(stg + r * PR + c0 + j) = q;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) stg[(c0 + j) * PT + r] = v[j];
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
    const int mvalid = min(128, M - m0);
    const int nvalid = min(BN, N - n0);
    if constexpr (MODE == TC_EPI_BIAS_RELU) {
      // rows m0.. of out (row stride ldo): nvalid floats each
      const int v4 = nvalid / 4;  // N % 4 == 0 (checked by the dispatcher)
      for (int e = tid; e < (csplit ? 0 : mvalid * v4); e += kProducers) {
        const int rr = e / v4, q = e - rr * v4;
        *reinterpret_cast<float4*>(epi.out + static_cast<std::size_t>(m0 + rr) * epi.ldo + n0 + 4 * q) =
            *reinterpret_cast<const float4*>(stg + rr * PR + 4 * q);
      }
    } else {
      // out[(split*N + n)*ldo + m0 + ...]: one 128-float row per n
      const int m4 = mvalid / 4;
      for (int e = tid; e < nvalid * 32; e += kProducers) {
        const int n = e >> 5, q = e & 31;
        if (q < m4)
          *reinterpret_cast<float4*>(epi.out + (static_cast<std::size_t>(split) * N + n0 + n) * epi.ldo + m0 +
                                     4 * q) = *reinterpret_cast<const float4*>(stg + n * PT + 4 * q);
      }
    }
  }
  if constexpr (MODE == TC_EPI_BIAS_RELU) {
    if (csplit) {
      // Split-K across the cluster (grid.y = cluster.y = KS): every CTA
      // staged its partial tile; CTA rank q finishes rows [q*RB, (q+1)*RB)
      // by summing the KS partials in rank order through DSMEM (fixed order:
      // deterministic), then bias + ReLU and coalesced stores.
      tc::cluster_sync();
      if (warp < kMmaWarp) {
        const int KS = gridDim.y;
        const int rank = static_cast<int>(tc::cluster_rank());
        constexpr int PR = BN + 4;
        const int mvalid = min(128, M - m0);
        const int v4 = min(BN, N - n0) / 4;
        const int RB = (128 + KS - 1) / KS;
        const int r0 = rank * RB, r1 = min(mvalid, r0 + RB);
        const uint32_t base = tc::smem_u32(smem);
        for (int e = tid; e < (r1 - r0) * v4; e += kProducers) {
          const int rr = r0 + e / v4, q = e % v4;
          const uint32_t off = base + static_cast<uint32_t>((rr * PR + 4 * q) * 4);
          float4 a = tc::ld_dsmem4(tc::mapa(off, 0));
          for (int k = 1; k < KS; ++k) {
            const float4 b = tc::ld_dsmem4(tc::mapa(off, k));
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
          }
          const int c = 4 * q;
          a.x += bias_sh[c];
          a.y += bias_sh[c + 1];
          a.z += bias_sh[c + 2];
          a.w += bias_sh[c + 3];
          a.x = a.x < 0.f ? 0.f : a.x;
          a.y = a.y < 0.f ? 0.f : a.y;
          a.z = a.z < 0.f ? 0.f : a.z;
          a.w = a.w < 0.f ? 0.f : a.w;
          *reinterpret_cast<float4*>(epi.out + static_cast<std::size_t>(m0 + rr) * epi.ldo + n0 + c) = a;
        }
      }
      tc::cluster_sync();  // partial tiles stay readable until every rank is done
    }
  }
  TRACE(3);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
  TRACE(4);
}

// =========================================================== MN-major GEMM
// X tile: 32 pixels x 128 kk (hi, then lo or u8 staging).  D tile: per 4-row
// k group, BN/32 hi atoms followed by BN/32 lo atoms (N-concatenated).
template <typename TX, int BN, int CAP = 0>
struct MNShape {
  static constexpr bool X_LO = sizeof(TX) == 4;
  static constexpr int X_SBO = 4 * 512;
  static constexpr int A_BYTES = 32 * 128 * 4;
  static constexpr int A_STG = X_LO ? A_BYTES : 32 * 128;
  static constexpr int D_ATOMS = BN / 32;
  static constexpr int D_SBO = 2 * D_ATOMS * 512;
  static constexpr int B_BYTES = 32 * 2 * BN * 4;
  static constexpr int STAGE = A_BYTES + A_STG + B_BYTES;
  static constexpr int NS = pipe::ring_depth(CAP, STAGE);
  static_assert(pipe::stages_for(STAGE) >= 2, "tile too large for a 2-stage pipeline");
  static constexpr int SMEM = NS * STAGE + 1024;
  static constexpr int TMEM_COLS = TmemCols<2 * BN>::V;
  static constexpr int DV = BN / 4;
  static constexpr int BVEC = 32 * DV;
  static constexpr int BN_PER = (BVEC + kProducers - 1) / kProducers;
};

template <typename TX, int BN, int CAP = 0>
__global__ void __launch_bounds__(kThreads, 1) tc_mn_ws_kernel(WgradArgs a) {
  static_assert(BN % 32 == 0 && 2 * BN <= 256, "MN-major tiles need 32-wide atoms, N <= 256");
  using S = MNShape<TX, BN, CAP>;
  constexpr int DV = S::DV;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t ready[pipe::kMaxStages], done[pipe::kMaxStages], acc_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_red[4 * kProducers];
  __shared__ float bias_cl[BN];  // cluster split: this rank's bias partials
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sbase = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kk0 = blockIdx.x * 128;
  const int n0 = blockIdx.z * BN;
  const int split = blockIdx.y;
  const int pb = split * a.kc;
  const int pe = min(a.npix, pb + a.kc);
  const int nchunks = (pe - pb + 31) / 32;
  const bool do_bias = blockIdx.x == 0 && a.mode == 0;
  // mode 1 with grid.y > 1: split-K over a (1, grid.y, 1) cluster
  const bool csplit = (a.mode == 1 || a.cluster) && gridDim.y > 1;

  const int xp = tid >> 3, xv = tid & 7;
  int xcoff[4];
  auto issue = [&](int c, uint32_t st) {
    const int pix = pb + 32 * c + xp;
    const bool pv = pix < pe;
    const int rb = pv ? a.X.rowbase(pix) : 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const bool ok = pv && xcoff[g] >= 0;
      if constexpr (sizeof(TX) == 4) {
        const float* src = static_cast<const float*>(a.X.p) + (ok ? rb + xcoff[g] + 4 * xv : 0);
        cp16(st + detail::mn_off(xp, g, xv, S::X_SBO), src, ok);
      } else {
        const uint8_t* src = static_cast<const uint8_t*>(a.X.p) + (ok ? rb + xcoff[g] + 4 * xv : 0);
        cp4(st + S::A_BYTES + xp * 128 + g * 32 + 4 * xv, src, ok);
      }
    }
    const uint32_t stb = st + S::A_BYTES + S::A_STG;
#pragma unroll
    for (int j = 0; j < S::BN_PER; ++j) {
      const int idx = tid + kProducers * j;
      if (idx >= S::BVEC) break;
      const int p = idx / DV, v = idx % DV;
      const int px = pb + 32 * c + p;
      const int co = n0 + 4 * v;
      const bool ok = px < pe && co < a.cout;
      const float* src = a.D + (ok ? static_cast<std::size_t>(px) * a.ldd + co : 0);
      cp16(stb + detail::mn_off(p, v >> 3, v & 7, S::D_SBO), src, ok);
    }
  };

  float4 bsum[S::BN_PER];
  TRACE(0);
  pdl_trigger();
  if (warp < kMmaWarp) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int kk = kk0 + 32 * g;
      xcoff[g] = kk < a.Kw ? a.X.chunkoff(kk) : -1;
    }
    pdl_wait();
#pragma unroll
    for (int c = 0; c < S::NS - 1; ++c) {
      if (c < nchunks) issue(c, sbase + c * S::STAGE);
      commit();
    }
  } else {
    tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S::NS; ++s) {
        tc::mbar_init(&ready[s], kProducers);
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
  TRACE(1);

  if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t id_cat = tc::idesc_tf32(128, 2 * BN, true, true);
      constexpr uint32_t id_one = tc::idesc_tf32(128, BN, true, true);
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % S::NS;
        tc::mbar_wait(&ready[s], (i / S::NS) & 1);
#ifdef GA3C_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_trace[8 + 2 * i] = t_;
        }
#endif
        tc::tc_fence_after();
        const uint32_t st = sbase + s * S::STAGE;
        const uint32_t a_hi = st, a_lo = st + S::A_BYTES, b = st + S::A_BYTES + S::A_STG;
#pragma unroll
        for (int h = 0; h < 4; ++h) {  // 8 pixels = two 4-row k groups per MMA
          const uint64_t dah = tc::sdesc(a_hi + 2 * h * S::X_SBO, 512, S::X_SBO, 1);
          const uint64_t db = tc::sdesc(b + 2 * h * S::D_SBO, 512, S::D_SBO, 1);
          tc::mma_tf32(tmem, dah, db, id_cat, (i | h) != 0);
          if constexpr (S::X_LO)
            tc::mma_tf32(tmem, tc::sdesc(a_lo + 2 * h * S::X_SBO, 512, S::X_SBO, 1), db, id_one, 1);
        }
        tc::mma_commit(&done[s]);
#ifdef GA3C_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_trace[9 + 2 * i] = t_;
        }
#endif
      }
      tc::mma_commit(&acc_bar);
    }
  } else {
#pragma unroll
    for (int j = 0; j < S::BN_PER; ++j) bsum[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % S::NS;
      const uint32_t st = sbase + s * S::STAGE;
      const uint32_t a_hi = st, a_lo = st + S::A_BYTES, b = st + S::A_BYTES + S::A_STG;
      wait_group<S::NS - 2>();
      TRACE(64 + 4 * i);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint32_t off = detail::mn_off(xp, g, xv, S::X_SBO);
        if constexpr (sizeof(TX) == 4)
          detail::sts128(a_lo + off, lo4(lds128(a_hi + off)));
        else
          detail::sts128(a_hi + off, widen_u8(lds32(a_lo + xp * 128 + g * 32 + 4 * xv)));
      }
#pragma unroll
      for (int j = 0; j < S::BN_PER; ++j) {
        const int idx = tid + kProducers * j;
        if (idx >= S::BVEC) break;
        const int p = idx / DV, v = idx % DV;
        const float4 d = lds128(b + detail::mn_off(p, v >> 3, v & 7, S::D_SBO));
        if (do_bias) {
          bsum[j].x += d.x;
          bsum[j].y += d.y;
          bsum[j].z += d.z;
          bsum[j].w += d.w;
        }
        detail::sts128(b + detail::mn_off(p, S::D_ATOMS + (v >> 3), v & 7, S::D_SBO), lo4(d));
      }
      tc::fence_async_smem();
      mbar_arrive(&ready[s]);
      const int nc = i + S::NS - 1;
      if (nc < nchunks) {
        const int ps = nc % S::NS;
        if (i >= 1) tc::mbar_wait(&done[ps], ((i - 1) / S::NS) & 1);
        issue(nc, sbase + ps * S::STAGE);
      }
      commit();
    }
    // ---- epilogue: C'[kk][co] staged transposed in smem as [co][kk], then
    // each warp writes whole 128-kk rows (512 B) with float4 stores
    TRACE(5);
    // mode 1: the ReLU gates of this warp's output rows, loaded while the
    // last MMAs drain (one round trip instead of one per row)
    constexpr int RPW = BN / (kProducers / 32);
    const int kvalid = min(128, a.Kw - kk0);  // multiple of 32 (Kw % 32 == 0)
    const bool lane_ok = 4 * lane < kvalid;
    // output rows this CTA finishes: all of them, or (cluster split-K) the
    // rank's block of BN / KS rows
    int rbase = 0, nco = min(BN, a.cout - n0);
    if (csplit) {
      const int RB = (BN + gridDim.y - 1) / gridDim.y;
      rbase = static_cast<int>(tc::cluster_rank()) * RB;
      nco = min(nco, rbase + RB);
    }
    float4 gts[RPW];
    if (a.mode == 1) {
#pragma unroll
      for (int j = 0; j < RPW; ++j) {
        const int row = rbase + warp + (kProducers / 32) * j;
        gts[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < nco && lane_ok)
          gts[j] = __ldg(reinterpret_cast<const float4*>(
              a.gate + static_cast<std::size_t>(n0 + row) * a.ldo + kk0 + 4 * lane));
      }
    }
    if (nchunks > 0) tc::mbar_wait(&acc_bar, 0);
    tc::tc_fence_after();
    TRACE(2);
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    constexpr int HALF = BN / 2;
    const int cbeg = (warp >> 2) * HALF;
    constexpr int PT = 128 + 4;
    float* stg = reinterpret_cast<float*>(smem);
    const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < HALF; c += 16) {
      const int c0 = cbeg + c;
      float v[16];
      if (nchunks > 0) {
        float w[16];
        tc::tmem_ld16(trow + c0, v);
        tc::tmem_ld16(trow + BN + c0, w);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w[j];
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) stg[(c0 + j) * PT + r] = v[j];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
    if (csplit) tc::cluster_sync();  // every rank's partial tile is staged
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int row = rbase + warp + (kProducers / 32) * j;
      if (row >= nco) break;
      const int co = n0 + row;
      float4 x;
      if (csplit) {
        // fixed rank order through DSMEM: deterministic
        x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (lane_ok) {
          const uint32_t off = tc::smem_u32(stg + row * PT + 4 * lane);
          x = tc::ld_dsmem4(tc::mapa(off, 0));
          for (int k = 1; k < static_cast<int>(gridDim.y); ++k) {
            const float4 y = tc::ld_dsmem4(tc::mapa(off, k));
            x.x += y.x;
            x.y += y.y;
            x.z += y.z;
            x.w += y.w;
          }
        }
      } else {
        x = *reinterpret_cast<const float4*>(stg + row * PT + 4 * lane);
      }
      if (a.mode == 1) {
        if (lane_ok) {
          const std::size_t o = static_cast<std::size_t>(co) * a.ldo + kk0 + 4 * lane;
          const float4 gt = gts[j];
          float4 y;
          y.x = gt.x <= 0.f ? 0.f : x.x;
          y.y = gt.y <= 0.f ? 0.f : x.y;
          y.z = gt.z <= 0.f ? 0.f : x.z;
          y.w = gt.w <= 0.f ? 0.f : x.w;
          *reinterpret_cast<float4*>(a.out + o) = y;
        }
      } else if (a.direct) {
        bool bad = false;
        if (lane_ok) {
          *reinterpret_cast<float4*>(a.gm.dtheta + a.gm.w0 + static_cast<std::size_t>(co) * a.Kw + kk0 + 4 * lane) = x;
          bad = !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.gm.flag, 1);
      } else if (lane_ok) {
        *reinterpret_cast<float4*>(a.part + (static_cast<std::size_t>(split) * a.cout + co) * a.Kw + kk0 +
                                   4 * lane) = x;
      }
    }
    TRACE(6);
    if (do_bias) {
      constexpr int R = kProducers / DV;
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
      asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");  // producer warps only
      if (tid < BN) {
        float sacc = 0.f;
        for (int r = 0; r < R; ++r) sacc += bias_red[r * BN + tid];
        const int co = n0 + tid;
        if (csplit) {
          bias_cl[tid] = sacc;  // reduced across the cluster below
        } else if (co < a.cout) {
          if (a.direct)
            a.gm.store(co, a.Kw, sacc);
          else
            a.part[static_cast<std::size_t>(gridDim.y) * a.cout * a.Kw + static_cast<std::size_t>(split) * a.cout +
                 co] = sacc;
        }
      }
    }
  }
  if (csplit) {
    // MMA warp: matches the producers' "staged" barrier; everyone: partial
    // tiles stay readable until every rank is done
    if (warp == kMmaWarp) tc::cluster_sync();
    tc::cluster_sync();
    if (a.mode == 0 && blockIdx.x == 0) {
      // bias column: rank 0 sums the ranks' partials in rank order
      if (tc::cluster_rank() == 0 && tid < BN && n0 + tid < a.cout) {
        const uint32_t off = tc::smem_u32(bias_cl + tid);
        float t = 0.f;
        for (int k = 0; k < static_cast<int>(gridDim.y); ++k) {
          float y;
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(y) : "r"(tc::mapa(off, k)) : "memory");
          t += y;
        }
        a.gm.store(n0 + tid, a.Kw, t);
      }
      tc::cluster_sync();  // the ranks' bias partials stay readable until read
    }
  }
  TRACE(3);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
  TRACE(4);
}

}  // namespace ws
}  // namespace ga3c
