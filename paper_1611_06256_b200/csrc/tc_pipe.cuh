// tc_pipe.cuh -- multi-stage cp.async pipelines feeding tcgen05 (kind::tf32).
//
// The tensor core reads an fp32 operand by TRUNCATING it to tf32 (measured on
// B200, tools/tc_probe.cu).  So the raw fp32 bytes, copied global->shared
// with cp.async straight into the 128B-swizzled canonical layout, already
// are the "hi" operand; only lo = x - trunc_tf32(x) is computed (smem->smem)
// and the 3xTF32 product A_hi*B_hi + A_hi*B_lo + A_lo*B_hi is issued as
// before.  u8 frames are staged raw and widened to f32 (exact, no lo).
// S stages of loads are in flight, so the per-chunk cost is the conversion +
// MMA issue instead of a global-memory round trip.
//
//   tc_kk_pipe_kernel : C[m][n] = sum_k A(m,k) B(n,k), both K-major (conv /
//                       FC forward; same Seg / epilogue contract as
//                       tc_kk_gemm_kernel)
//   tc_mn_pipe_kernel : C'[kk][co] = sum_m X(m,kk) D(m,co), both MN-major
//                       (weight gradients and the transposed FC input
//                       gradient; same WgradArgs contract as tc_wgrad_kernel)
#pragma once

#include <cstdint>

#include "tc_common.cuh"
#include "tc_gemm.cuh"
#include "tc_wgrad.cuh"

#ifdef GA3C_TRACE
__device__ unsigned long long g_trace[256];
#define TRACE(i)                                                                              \
  do {                                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) {          \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      g_trace[i] = t_;                                                                        \
    }                                                                                         \
  } while (0)
#else
#define TRACE(i) \
  do {           \
  } while (0)
#endif

namespace ga3c {
namespace pipe {

constexpr int kMaxStages = 8;
constexpr int stages_for(int stage_bytes) {
  return (220 * 1024) / stage_bytes < kMaxStages ? (220 * 1024) / stage_bytes : kMaxStages;
}
// Ring depth for a stage cap: 0 = as deep as ~220 KB of shared memory
// allows (one CTA per SM), 1 = at most ~100 KB (two CTAs per SM: a
// multi-wave grid, or CTAs of concurrent kernels, share the SM), n >= 2 = at
// most n stages (a CTA that only ever streams n chunks needs no more; the
// smaller footprint lets other kernels' CTAs co-reside).  Never below 2.
constexpr int ring_depth(int cap, int stage_bytes) {
  const int deep = stages_for(stage_bytes);
  const int two = (100 * 1024) / stage_bytes;  // + static smem and alignment: two CTAs fit in 228 KB
  const int d = cap == 0 ? deep : (cap == 1 ? (two < deep ? two : deep) : (cap < deep ? cap : deep));
  return d < 2 ? 2 : d;
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ float lo_of(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ float4 lo4(float4 x) {
  return make_float4(lo_of(x.x), lo_of(x.y), lo_of(x.z), lo_of(x.w));
}

// byte i of w as the fp32 2^23 + byte (PRMT against 0x4B000000): no I2F,
// which issues on the quarter-rate XU pipe
__device__ __forceinline__ float magic_u8(uint32_t w, uint32_t sel) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, sel));
}

// four u8 frame bytes -> fp32 x / 256, exactly: (2^23 + x) * 2^-8 - 2^15 is
// one FFMA with an exact product and an exact result
__device__ __forceinline__ float4 widen_u8(uint32_t w) {
  float4 f;
  f.x = __fmaf_rn(magic_u8(w, 0x7650u), 1.0f / 256.0f, -32768.0f);
  f.y = __fmaf_rn(magic_u8(w, 0x7651u), 1.0f / 256.0f, -32768.0f);
  f.z = __fmaf_rn(magic_u8(w, 0x7652u), 1.0f / 256.0f, -32768.0f);
  f.w = __fmaf_rn(magic_u8(w, 0x7653u), 1.0f / 256.0f, -32768.0f);
  return f;
}

// ------------------------------------------------------------ K-major tiles
// ROWS x 32 k of a K-major operand.  f32: cp.async 16 B vectors into the
// swizzled hi tile, lo computed in place.  u8: cp.async 4 B words into a
// linear staging area [ROWS][32 B], widened into the swizzled f32 tile.
template <typename T, int ROWS>
struct KTile;

template <int ROWS>
struct KTile<float, ROWS> {
  static constexpr int VEC = ROWS * 8;
  static constexpr int N = (VEC + kTcThreads - 1) / kTcThreads;
  static constexpr int HI_BYTES = ROWS * 128;
  static constexpr int BYTES = 2 * HI_BYTES;  // hi + lo
  int goff[N];
  uint32_t soff[N];
  __device__ __forceinline__ void init(const Seg& s, int row0, int tid) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int idx = tid + kTcThreads * j;
      const int r = idx >> 3, v = idx & 7;
      const int g = row0 + r;
      goff[j] = (idx < VEC && g < s.rows) ? s.rowbase(g) + 4 * v : -1;
      soff[j] = tc::sw128_off(r, v);
    }
  }
  __device__ __forceinline__ void issue(const Seg& s, int coff, uint32_t base, int tid) const {
    const float* src = static_cast<const float*>(s.p) + coff;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (tid + kTcThreads * j >= VEC) break;
      cp16(base + soff[j], src + (goff[j] >= 0 ? goff[j] : 0), goff[j] >= 0);
    }
  }
  __device__ __forceinline__ void convert(uint32_t base, int tid) const {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (tid + kTcThreads * j >= VEC) break;
      detail::sts128(base + HI_BYTES + soff[j], lo4(lds128(base + soff[j])));
    }
  }
  __device__ __forceinline__ uint32_t hi(uint32_t base) const { return base; }
  __device__ __forceinline__ uint32_t lo(uint32_t base) const { return base + HI_BYTES; }
};

template <int ROWS>
struct KTile<uint8_t, ROWS> {
  static constexpr int VEC = ROWS * 8;  // 4-byte words
  static constexpr int N = (VEC + kTcThreads - 1) / kTcThreads;
  static constexpr int HI_BYTES = ROWS * 128;
  static constexpr int STG_BYTES = ROWS * 32;
  static constexpr int BYTES = HI_BYTES + STG_BYTES;
  int goff[N];
  uint32_t soff[N];
  __device__ __forceinline__ void init(const Seg& s, int row0, int tid) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int idx = tid + kTcThreads * j;
      const int r = idx >> 3, q = idx & 7;
      const int g = row0 + r;
      goff[j] = (idx < VEC && g < s.rows) ? s.rowbase(g) + 4 * q : -1;
      soff[j] = tc::sw128_off(r, q);
    }
  }
  __device__ __forceinline__ void issue(const Seg& s, int coff, uint32_t base, int tid) const {
    const uint8_t* src = static_cast<const uint8_t*>(s.p) + coff;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int idx = tid + kTcThreads * j;
      if (idx >= VEC) break;
      cp4(base + HI_BYTES + 4 * idx, src + (goff[j] >= 0 ? goff[j] : 0), goff[j] >= 0);
    }
  }
  __device__ __forceinline__ void convert(uint32_t base, int tid) const {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int idx = tid + kTcThreads * j;
      if (idx >= VEC) break;
      detail::sts128(base + soff[j], widen_u8(lds32(base + HI_BYTES + 4 * idx)));
    }
  }
  __device__ __forceinline__ uint32_t hi(uint32_t base) const { return base; }
  __device__ __forceinline__ uint32_t lo(uint32_t base) const { return base; }
};

template <typename TA, typename TB, int BN>
struct KKPipeShape {
  using TileA = KTile<TA, 128>;
  using TileB = KTile<TB, BN>;
  static constexpr int STAGE = TileA::BYTES + TileB::BYTES;
  static constexpr int NS = stages_for(STAGE);
  static_assert(NS >= 2, "tile too large for a 2-stage pipeline");
  static constexpr int SMEM = NS * STAGE + 1024;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

template <typename TA, typename TB, int BN, int MODE>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_kk_pipe_kernel(Seg A, Seg B, int M, int N, int K, int kc, TcEpiArgs epi) {
  using S = KKPipeShape<TA, TB, BN>;
  constexpr bool A_LO = sizeof(TA) == 4, B_LO = sizeof(TB) == 4;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bars[kMaxStages];
  __shared__ uint32_t tmem_base_sh;
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sbase = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.z * BN;
  const int split = blockIdx.y;
  const int kb = split * kc;
  const int ke = min(K, kb + kc);
  const int nchunks = (ke - kb + 31) / 32;

  TRACE(0);
  typename S::TileA ta;
  typename S::TileB tb;
  ta.init(A, m0, tid);
  tb.init(B, n0, tid);
  TRACE(5);
  // prologue: S-1 chunks in flight
#pragma unroll
  for (int c = 0; c < S::NS - 1; ++c) {
    if (c < nchunks) {
      const uint32_t st = sbase + c * S::STAGE;
      ta.issue(A, A.chunkoff(kb + 32 * c), st, tid);
      tb.issue(B, B.chunkoff(kb + 32 * c), st + S::TileA::BYTES, tid);
    }
    commit();
  }
  TRACE(6);
  if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
  TRACE(7);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S::NS; ++s) tc::mbar_init(&bars[s], 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t idesc = tc::idesc_tf32(128, BN, false, false);
  TRACE(1);

  for (int i = 0; i < nchunks; ++i) {
    const int s = i % S::NS;
    const uint32_t st = sbase + s * S::STAGE;
    const uint32_t stb = st + S::TileA::BYTES;
    wait_group<S::NS - 2>();
    __syncthreads();  // chunk i resident for every thread
    TRACE(8 + 2 * i);
    ta.convert(st, tid);
    tb.convert(stb, tid);
    TRACE(64 + 4 * i);
    tc::fence_async_smem();
    TRACE(65 + 4 * i);
    __syncthreads();
    TRACE(66 + 4 * i);
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t ah = ta.hi(st), al = ta.lo(st), bh = tb.hi(stb), bl = tb.lo(stb);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t dah = tc::sdesc_sw128(ah + kk * 32, 16, 1024);
        const uint64_t dbh = tc::sdesc_sw128(bh + kk * 32, 16, 1024);
        tc::mma_tf32(tmem, dah, dbh, idesc, (i | kk) != 0);
        if constexpr (B_LO) tc::mma_tf32(tmem, dah, tc::sdesc_sw128(bl + kk * 32, 16, 1024), idesc, 1);
        if constexpr (A_LO) tc::mma_tf32(tmem, tc::sdesc_sw128(al + kk * 32, 16, 1024), dbh, idesc, 1);
      }
      tc::mma_commit(&bars[s]);
    }
    TRACE(9 + 2 * i);
    // refill the stage chunk i-1 used, once its MMAs have drained
    const int nc = i + S::NS - 1;
    if (nc < nchunks) {
      const int ps = nc % S::NS;
      if (i >= 1) tc::mbar_wait(&bars[ps], ((i - 1) / S::NS) & 1);
      const uint32_t pst = sbase + ps * S::STAGE;
      ta.issue(A, A.chunkoff(kb + 32 * nc), pst, tid);
      tb.issue(B, B.chunkoff(kb + 32 * nc), pst + S::TileA::BYTES, tid);
    }
    commit();
  }
  const int last = nchunks - 1;
  if (nchunks > 0) tc::mbar_wait(&bars[last % S::NS], (last / S::NS) & 1);
  tc::tc_fence_after();
  TRACE(2);

  const int quad = warp & 3;
  const int row = quad * 32 + lane;
  const int m = m0 + row;
  constexpr int HALF = BN >= 32 ? BN / 2 : BN;
  const int cbeg = (warp >> 2) * HALF;
  if (cbeg < BN) {
#pragma unroll 1
    for (int c = 0; c < HALF; c += 16) {
      const int c0 = cbeg + c;
      float v[16];
      tc::tmem_ld16(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0, v);
      tc::tmem_ld_wait();
      if (m < M) {
        if constexpr (MODE == TC_EPI_BIAS_RELU) {
          float* o = epi.out + static_cast<std::size_t>(m) * epi.ldo + n0 + c0;
          if (n0 + c0 + 16 <= N) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const float* bp = epi.bias + n0 + c0 + j;
              float4 r;
              r.x = v[j] + __ldg(bp);
              r.y = v[j + 1] + __ldg(bp + 1);
              r.z = v[j + 2] + __ldg(bp + 2);
              r.w = v[j + 3] + __ldg(bp + 3);
              r.x = r.x < 0.f ? 0.f : r.x;
              r.y = r.y < 0.f ? 0.f : r.y;
              r.z = r.z < 0.f ? 0.f : r.z;
              r.w = r.w < 0.f ? 0.f : r.w;
              *reinterpret_cast<float4*>(o + j) = r;
            }
          } else {
            for (int j = 0; j < 16 && n0 + c0 + j < N; ++j) {
              const float r = v[j] + __ldg(epi.bias + n0 + c0 + j);
              o[j] = r < 0.f ? 0.f : r;
            }
          }
        } else {
          float* o = epi.out + (static_cast<std::size_t>(split) * N + n0 + c0) * epi.ldo + m;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (n0 + c0 + j < N) o[static_cast<std::size_t>(j) * epi.ldo] = v[j];
        }
      }
    }
  }
  TRACE(3);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
  TRACE(4);
}

// ----------------------------------------------------------- MN-major tiles
// 32 k-rows (pixels) x E MN elements in the SWIZZLE_128B_BASE32B layout
// (tc_wgrad.cuh detail::mn_off): MN atoms of 32 at 512 B (LBO), 4-row k
// groups at SBO = (E/32)*512.
template <int E>
struct MnGeom {
  static constexpr int SBO = (E / 32) * 512;
  static constexpr int BYTES = 32 * E * 4;
};

template <typename TX, int BN>
struct MnPipeShape {
  static constexpr bool X_LO = sizeof(TX) == 4;
  static constexpr int A_BYTES = MnGeom<128>::BYTES;        // 16 KB
  static constexpr int A_STG = X_LO ? A_BYTES : 32 * 128;   // lo tile or u8 staging
  static constexpr int B_BYTES = MnGeom<BN>::BYTES;
  static constexpr int STAGE = A_BYTES + A_STG + 2 * B_BYTES;
  static constexpr int NS = stages_for(STAGE);
  static_assert(NS >= 2, "tile too large for a 2-stage pipeline");
  static constexpr int SMEM = NS * STAGE + 1024;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int DV = BN / 4;
  static constexpr int BVEC = 32 * DV;
  static constexpr int BN_PER = (BVEC + kTcThreads - 1) / kTcThreads;
};

template <typename TX, int BN>
__global__ void __launch_bounds__(kTcThreads, 1) tc_mn_pipe_kernel(WgradArgs a) {
  static_assert(BN % 32 == 0, "MN-major needs 32-wide N atoms");
  using S = MnPipeShape<TX, BN>;
  constexpr int DV = S::DV;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bars[kMaxStages];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_red[4 * kTcThreads];
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

  // X tile: thread -> (pixel row xp, vector xv) x 4 kk atoms
  const int xp = tid >> 3, xv = tid & 7;
  int xcoff[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int kk = kk0 + 32 * g;
    xcoff[g] = kk < a.Kw ? a.X.chunkoff(kk) : -1;
  }
  auto issue = [&](int c, uint32_t st) {
    const int pix = pb + 32 * c + xp;
    const bool pv = pix < pe;
    const int rb = pv ? a.X.rowbase(pix) : 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const bool ok = pv && xcoff[g] >= 0;
      if constexpr (sizeof(TX) == 4) {
        const float* src = static_cast<const float*>(a.X.p) + (ok ? rb + xcoff[g] + 4 * xv : 0);
        cp16(st + detail::mn_off(xp, g, xv, MnGeom<128>::SBO), src, ok);
      } else {
        const uint8_t* src = static_cast<const uint8_t*>(a.X.p) + (ok ? rb + xcoff[g] + 4 * xv : 0);
        cp4(st + S::A_BYTES + xp * 128 + g * 32 + 4 * xv, src, ok);
      }
    }
    const uint32_t stb = st + S::A_BYTES + S::A_STG;
#pragma unroll
    for (int j = 0; j < S::BN_PER; ++j) {
      const int idx = tid + kTcThreads * j;
      if (idx >= S::BVEC) break;
      const int p = idx / DV, v = idx % DV;
      const int px = pb + 32 * c + p;
      const int co = n0 + 4 * v;
      const bool ok = px < pe && co < a.cout;
      const float* src = a.D + (ok ? static_cast<std::size_t>(px) * a.ldd + co : 0);
      cp16(stb + detail::mn_off(p, v >> 3, v & 7, MnGeom<BN>::SBO), src, ok);
    }
  };

#pragma unroll
  for (int c = 0; c < S::NS - 1; ++c) {
    if (c < nchunks) issue(c, sbase + c * S::STAGE);
    commit();
  }
  if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S::NS; ++s) tc::mbar_init(&bars[s], 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t idesc = tc::idesc_tf32(128, BN, true, true);
  float4 bsum[S::BN_PER];
#pragma unroll
  for (int j = 0; j < S::BN_PER; ++j) bsum[j] = make_float4(0.f, 0.f, 0.f, 0.f);

  for (int i = 0; i < nchunks; ++i) {
    const int s = i % S::NS;
    const uint32_t st = sbase + s * S::STAGE;
    const uint32_t a_hi = st, a_lo = st + S::A_BYTES;
    const uint32_t b_hi = st + S::A_BYTES + S::A_STG, b_lo = b_hi + S::B_BYTES;
    wait_group<S::NS - 2>();
    __syncthreads();
    // X: lo tile (f32) or widen the u8 staging into the f32 tile
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint32_t off = detail::mn_off(xp, g, xv, MnGeom<128>::SBO);
      if constexpr (sizeof(TX) == 4)
        detail::sts128(a_lo + off, lo4(lds128(a_hi + off)));
      else
        detail::sts128(a_hi + off, widen_u8(lds32(a_lo + xp * 128 + g * 32 + 4 * xv)));
    }
    // D: lo tile (+ bias column sums)
#pragma unroll
    for (int j = 0; j < S::BN_PER; ++j) {
      const int idx = tid + kTcThreads * j;
      if (idx >= S::BVEC) break;
      const int p = idx / DV, v = idx % DV;
      const uint32_t off = detail::mn_off(p, v >> 3, v & 7, MnGeom<BN>::SBO);
      const float4 d = lds128(b_hi + off);
      if (do_bias) {
        bsum[j].x += d.x;
        bsum[j].y += d.y;
        bsum[j].z += d.z;
        bsum[j].w += d.w;
      }
      detail::sts128(b_lo + off, lo4(d));
    }
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint64_t dah = tc::sdesc(a_hi + 2 * h * MnGeom<128>::SBO, 512, MnGeom<128>::SBO, 1);
        const uint64_t dbh = tc::sdesc(b_hi + 2 * h * MnGeom<BN>::SBO, 512, MnGeom<BN>::SBO, 1);
        tc::mma_tf32(tmem, dah, dbh, idesc, (i | h) != 0);
        tc::mma_tf32(tmem, dah, tc::sdesc(b_lo + 2 * h * MnGeom<BN>::SBO, 512, MnGeom<BN>::SBO, 1),
                     idesc, 1);
        if constexpr (S::X_LO)
          tc::mma_tf32(tmem, tc::sdesc(a_lo + 2 * h * MnGeom<128>::SBO, 512, MnGeom<128>::SBO, 1), dbh,
                       idesc, 1);
      }
      tc::mma_commit(&bars[s]);
    }
    const int nc = i + S::NS - 1;
    if (nc < nchunks) {
      const int ps = nc % S::NS;
      if (i >= 1) tc::mbar_wait(&bars[ps], ((i - 1) / S::NS) & 1);
      issue(nc, sbase + ps * S::STAGE);
    }
    commit();
  }
  const int last = nchunks - 1;
  if (nchunks > 0) tc::mbar_wait(&bars[last % S::NS], (last / S::NS) & 1);
  tc::tc_fence_after();

  const int quad = warp & 3;
  const int row = quad * 32 + lane;
  const int kk = kk0 + row;
  constexpr int HALF = BN / 2;
  const int cbeg = (warp >> 2) * HALF;
  const int ldp = a.Kw + 1;
#pragma unroll 1
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
#pragma unroll 4
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

}  // namespace pipe
}  // namespace ga3c
