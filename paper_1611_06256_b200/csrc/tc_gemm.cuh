// tc_gemm.cuh -- tcgen05 implicit GEMM for the GA3C trunk contractions.
//
//   C[m][n] = sum_k A(m,k) * B(n,k)      (both operands K-major)
//
// One CTA (8 warps) owns a 128-row M tile and a BN-column N tile; the
// accumulator lives in TMEM (128 lanes x BN fp32 columns).  Operand tiles are
// gathered by all warps straight from the NHWC activations / u8 frames
// (implicit im2col: every (row, 32-wide k chunk) is one contiguous run), split
// into tf32 hi/lo halves and written to shared memory in the 128B-swizzled
// K-major canonical layout; one thread issues
//   A_hi*B_hi + A_hi*B_lo + A_lo*B_hi          (3xTF32, ~fp32 accuracy)
// per 8-deep k-step (the lo terms vanish for u8 frames, exact in tf32).  The
// next chunk's global loads are in flight while the current chunk is
// multiplied (double-buffered smem, tcgen05.commit -> mbarrier).  Row
// offsets and swizzled smem offsets are computed once per CTA, so the gather
// costs ~2 instructions per 16-byte vector.  Split-K over blockIdx.y writes
// partial sums that a fixed-order reduction consumes (deterministic).
#pragma once

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

// x = hi + lo: hi = x with the low 13 mantissa bits cleared (exactly tf32),
// lo = x - hi exactly; the MMA reads lo's top 11 significant bits, so
// hi*b + lo*b reproduces x*b to ~2^-21 relative.
__device__ __forceinline__ void split1(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

// One 32-wide k chunk of a ROWS-row tile, as per-thread registers.
template <typename T, int ROWS>
struct Chunk;

template <int ROWS>
struct Chunk<float, ROWS> {
  static constexpr int VEC = ROWS * 8;  // 16-byte vectors per chunk
  static constexpr int N = (VEC + kTcThreads - 1) / kTcThreads;
  int goff[N];       // element offset of this thread's vector (without chunk), -1 = zero
  uint32_t soff[N];  // swizzled smem byte offset
  float4 x[N];
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
  __device__ __forceinline__ void load(const Seg& s, int coff) {
    const float* base = static_cast<const float*>(s.p) + coff;
#pragma unroll
    for (int j = 0; j < N; ++j)
      x[j] = goff[j] >= 0 ? __ldg(reinterpret_cast<const float4*>(base + goff[j]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  template <bool LO>
  __device__ __forceinline__ void store(uint32_t hi, uint32_t lo, int tid) const {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (tid + kTcThreads * j >= VEC) break;
      float4 h, l;
      split1(x[j].x, h.x, l.x);
      split1(x[j].y, h.y, l.y);
      split1(x[j].z, h.z, l.z);
      split1(x[j].w, h.w, l.w);
      sts128(hi + soff[j], h);
      if constexpr (LO) sts128(lo + soff[j], l);
    }
  }
};

// u8 frames: x = k/256 is exact in tf32 -> no lo half.  Runs are read as
// 4-byte words (only 4-byte alignment is needed, e.g. stride-1 conv1).
template <int ROWS>
struct Chunk<uint8_t, ROWS> {
  static constexpr int VEC = ROWS * 8;  // 4-byte words per chunk
  static constexpr int N = (VEC + kTcThreads - 1) / kTcThreads;
  int goff[N];
  uint32_t soff[N];
  uint32_t w[N];
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
  __device__ __forceinline__ void load(const Seg& s, int coff) {
    const uint8_t* base = static_cast<const uint8_t*>(s.p) + coff;
#pragma unroll
    for (int j = 0; j < N; ++j)
      w[j] = goff[j] >= 0 ? __ldg(reinterpret_cast<const uint32_t*>(base + goff[j])) : 0u;
  }
  template <bool LO>
  __device__ __forceinline__ void store(uint32_t hi, uint32_t, int tid) const {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (tid + kTcThreads * j >= VEC) break;
      float4 f;
      f.x = static_cast<float>(w[j] & 0xFFu) * (1.0f / 256.0f);
      f.y = static_cast<float>((w[j] >> 8) & 0xFFu) * (1.0f / 256.0f);
      f.z = static_cast<float>((w[j] >> 16) & 0xFFu) * (1.0f / 256.0f);
      f.w = static_cast<float>(w[j] >> 24) * (1.0f / 256.0f);
      sts128(hi + soff[j], f);
    }
  }
};

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

template <typename TA, typename TB, int BN, int MODE>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_kk_gemm_kernel(Seg A, Seg B, int M, int N, int K, int kc, TcEpiArgs epi) {
  using S = TcShape<TA, TB, BN>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem_base_sh;
  uint8_t* smem = detail::align1024(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.z * BN;
  const int split = blockIdx.y;
  const int kb = split * kc;
  const int ke = min(K, kb + kc);
  const int nchunks = (ke - kb + 31) / 32;

  detail::Chunk<TA, 128> ca;
  detail::Chunk<TB, BN> cb;
  ca.init(A, m0, tid);
  cb.init(B, n0, tid);
  if (nchunks > 0) {  // first loads fly during the TMEM / barrier setup
    ca.load(A, A.chunkoff(kb));
    cb.load(B, B.chunkoff(kb));
  }
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
  constexpr uint32_t idesc = tc::idesc_tf32(128, BN, false, false);

  for (int i = 0; i < nchunks; ++i) {
    const int s = i & 1;
    if (i >= 2) tc::mbar_wait(&bars[s], ((i >> 1) - 1) & 1);
    const uint32_t st = tc::smem_u32(smem + s * S::STAGE);
    const uint32_t a_hi = st;
    const uint32_t a_lo = st + S::A_BYTES;
    const uint32_t b_hi = st + S::A_BYTES * (S::A_LO ? 2 : 1);
    const uint32_t b_lo = b_hi + S::B_BYTES;
    ca.template store<S::A_LO>(a_hi, a_lo, tid);
    cb.template store<S::B_LO>(b_hi, b_lo, tid);
    if (i + 1 < nchunks) {  // next chunk's loads fly while this one is multiplied
      const int k1 = kb + 32 * (i + 1);
      ca.load(A, A.chunkoff(k1));
      cb.load(B, B.chunkoff(k1));
    }
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t dah = tc::sdesc_sw128(a_hi + kk * 32, 16, 1024);
        const uint64_t dbh = tc::sdesc_sw128(b_hi + kk * 32, 16, 1024);
        tc::mma_tf32(tmem, dah, dbh, idesc, (i | kk) != 0);
        if constexpr (S::B_LO) tc::mma_tf32(tmem, dah, tc::sdesc_sw128(b_lo + kk * 32, 16, 1024), idesc, 1);
        if constexpr (S::A_LO) tc::mma_tf32(tmem, tc::sdesc_sw128(a_lo + kk * 32, 16, 1024), dbh, idesc, 1);
      }
      tc::mma_commit(&bars[s]);
    }
  }
  const int last = nchunks - 1;
  tc::mbar_wait(&bars[last & 1], (last >> 1) & 1);
  tc::tc_fence_after();

  // epilogue: warp w reads TMEM lanes 32*(w%4).. (rows), column half w/4
  const int quad = warp & 3;
  const int row = quad * 32 + lane;
  const int m = m0 + row;
  constexpr int HALF = BN >= 32 ? BN / 2 : BN;
  const int cbeg = (warp >> 2) * HALF;
  if (cbeg < BN) {
#pragma unroll
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
              float4 r;
              r.x = v[j] + __ldg(epi.bias + n0 + c0 + j);
              r.y = v[j + 1] + __ldg(epi.bias + n0 + c0 + j + 1);
              r.z = v[j + 2] + __ldg(epi.bias + n0 + c0 + j + 2);
              r.w = v[j + 3] + __ldg(epi.bias + n0 + c0 + j + 3);
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
          // transposed partials: out[(split * N + n) * M + m]
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = n0 + c0 + j;
            if (n < N) epi.out[(static_cast<std::size_t>(split) * N + n) * epi.ldo + m] = v[j];
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace ga3c
