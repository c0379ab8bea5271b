// tc_bf16.cuh -- conv forward on raw u8 frames with tcgen05.mma kind::f16
// (bf16 operands, fp32 accumulate), exact to fp32 accuracy.
//
// A frame byte k is an 8-bit integer, exactly representable in bf16, so the
// A operand is the frame itself (the 1/256 input scale is a power of two and
// is applied to the fp32 accumulator in the epilogue: identical result).
// An fp32 weight w splits EXACTLY into three bf16 pieces by truncation,
//   hi = trunc16(w), mid = trunc16(w - hi), lo = w - hi - mid
// (24 significand bits = 3 x 8), and every product k * piece is exact in
// fp32.  The three pieces are N-concatenated ([W_hi; W_mid; W_lo], N = 3*BN)
// so one MMA per 16-wide k-step covers all of them; the epilogue sums the
// three accumulator ranges.  Compared with 3xTF32 on the widened frame this
// halves the MMA count (K = 16 per instruction instead of 8, one
// instruction instead of one per split term) and the A tile's shared-memory
// bytes, and drops no cross term.
//
// Same warp-specialized structure as tc_ws.cuh: 8 producer warps stage u8
// rows and fp32 weights with cp.async, convert them into 128B-swizzled
// K-major bf16 tiles and signal ready[]; one warp issues the MMAs; the
// producers run the epilogue (bias + ReLU, or cluster split-K through DSMEM).
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

#include "pdl.cuh"
#include "tc_pipe.cuh"

namespace ga3c {
namespace bf {

constexpr int kProducers = 256;
constexpr int kThreads = kProducers + 32;
constexpr int kMmaWarp = kProducers / 32;
constexpr int KC = 64;  // K elements per chunk (one 128-byte bf16 row)

// kind::f16 instruction descriptor: c_format F32 (1), a/b_format BF16 (1),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void lds64(uint32_t a, uint32_t& x, uint32_t& y) {
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
}

__device__ __forceinline__ void sts128u(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// two u8 (as integers) -> packed bf16x2 (exact).  float(b) = (2^23 + b) - 2^23
// via PRMT + FADD instead of I2F (quarter-rate XU pipe).
__device__ __forceinline__ uint32_t u8x2_bf16(uint32_t b0, uint32_t b1) {
  const uint32_t f0 = __float_as_uint(__uint_as_float(0x4B000000u | b0) - 8388608.0f);
  const uint32_t f1 = __float_as_uint(__uint_as_float(0x4B000000u | b1) - 8388608.0f);
  return __byte_perm(f0, f1, 0x7632);  // upper halves: exact truncation of small integers
}

// w = hi + mid + lo exactly, each a bf16 (returned as the upper 16 bits)
__device__ __forceinline__ void split3(float w, uint32_t& hi, uint32_t& mid, uint32_t& lo) {
  const uint32_t h = __float_as_uint(w) & 0xFFFF0000u;
  const float r1 = w - __uint_as_float(h);
  const uint32_t m = __float_as_uint(r1) & 0xFFFF0000u;
  const float r2 = r1 - __uint_as_float(m);
  hi = h;
  mid = m;
  lo = __float_as_uint(r2);
}

__device__ __forceinline__ float relu(float x) { return x < 0.f ? 0.f : x; }  // NaN passes, as elsewhere

__device__ __forceinline__ uint32_t pack_hi(uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x7632); }

template <int BN>
struct U8Shape {
  static constexpr int A_STG = 128 * KC;       // u8 staging, 64 B per row
  static constexpr int A_BYTES = 128 * 128;    // bf16 tile, SW128
  static constexpr int B_STG = BN * KC * 4;    // fp32 staging, 256 B per row
  static constexpr int B_BYTES = 3 * BN * 128; // [hi; mid; lo] bf16 rows, SW128
  static constexpr int STAGE = A_STG + A_BYTES + B_STG + B_BYTES;
  static constexpr int NS_DEEP = pipe::stages_for(STAGE);
  static constexpr int ACC_COLS = 3 * BN;
  static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : (ACC_COLS <= 64 ? 64 : (ACC_COLS <= 128 ? 128 : 256));
  static constexpr int AU_PER = 128 * 8 / kProducers;  // 16-byte bf16 units per thread
  static constexpr int BU = BN * 8;                    // 8-element units of W per chunk
  static constexpr int BU_PER = (BU + kProducers - 1) / kProducers;
};

// C[m][n] = ReLU(bias[n] + (1/256) * sum_k frame_u8(m, k) * W[n][k])
// A: im2col Seg over u8 NHWC frames (rowlen % 32 == 0); W: dense fp32 [N][K]
// (Seg with rows = N, rowlen = K); K % 64 == 0, BN in {16, 32, 64}.
template <int BN, int CAP>
__global__ void __launch_bounds__(kThreads, 1)
tc_u8_fwd_kernel(Seg A, Seg B, int M, int N, int K, int kc, TcEpiArgs epi) {
  using S = U8Shape<BN>;
  constexpr int NS = pipe::ring_depth(CAP, S::STAGE);
  static_assert(3 * BN <= 256 && BN % 16 == 0, "N-concatenated tile exceeds the MMA N limit");
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t ready[pipe::kMaxStages], done[pipe::kMaxStages], acc_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_sh[BN];
  uint8_t* smem = detail::align1024(smem_raw);
  const uint32_t sbase = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.z * BN;
  const int kb = blockIdx.y * kc;
  const int ke = min(K, kb + kc);
  const int nchunks = (ke - kb + KC - 1) / KC;
  const bool csplit = gridDim.y > 1;

  // Each producer thread converts exactly the bytes its own cp.asyncs
  // staged (wait_group only covers the calling thread's copies): A units of
  // 8 K-elements (two 4-byte words of one row) and W units of 8 floats.
  int arow_base[S::AU_PER];
  int bgoff[S::BU_PER];
  pdl_trigger();
  if (warp < kMmaWarp) {
#pragma unroll
    for (int j = 0; j < S::AU_PER; ++j) {
      const int u = tid + kProducers * j;
      const int g = m0 + (u >> 3);
      arow_base[j] = g < A.rows ? A.rowbase(g) : -1;
    }
#pragma unroll
    for (int j = 0; j < S::BU_PER; ++j) {
      const int u = tid + kProducers * j;
      const int g = n0 + (u >> 3);
      bgoff[j] = (u < S::BU && g < B.rows) ? B.rowbase(g) + 8 * (u & 7) : -1;
    }
  }
  auto issue = [&](int c, uint32_t st) {
    const int k0 = kb + KC * c;
    const int off0 = A.chunkoff(k0), off1 = A.chunkoff(k0 + 32);
    const uint8_t* ap = static_cast<const uint8_t*>(A.p);
#pragma unroll
    for (int j = 0; j < S::AU_PER; ++j) {
      const int u = tid + kProducers * j;
      const int r = u >> 3, q = u & 7;
      const int off = (q < 4 ? off0 : off1) + 8 * (q & 3);
      const bool ok = arow_base[j] >= 0;
      const uint8_t* src = ap + (ok ? arow_base[j] + off : 0);
      pipe::cp4(st + r * KC + 8 * q, src, ok);
      pipe::cp4(st + r * KC + 8 * q + 4, src + 4, ok);
    }
    const float* bp = static_cast<const float*>(B.p) + k0;
    const uint32_t bst = st + S::A_STG + S::A_BYTES;
#pragma unroll
    for (int j = 0; j < S::BU_PER; ++j) {
      const int u = tid + kProducers * j;
      if (u >= S::BU) break;
      const bool ok = bgoff[j] >= 0;
      const float* src = bp + (ok ? bgoff[j] : 0);
      pipe::cp16(bst + (u >> 3) * 256 + 32 * (u & 7), src, ok);
      pipe::cp16(bst + (u >> 3) * 256 + 32 * (u & 7) + 16, src + 4, ok);
    }
  };
  auto convert = [&](uint32_t st) {
    // A: u8 row-major [128][64] -> bf16 SW128 [128][128 B]
#pragma unroll
    for (int j = 0; j < S::AU_PER; ++j) {
      const int u = tid + kProducers * j;
      const int r = u >> 3, q = u & 7;
      uint32_t x, y;
      lds64(st + r * KC + 8 * q, x, y);
      sts128u(st + S::A_STG + tc::sw128_off(r, q), u8x2_bf16(x & 0xFF, (x >> 8) & 0xFF),
              u8x2_bf16((x >> 16) & 0xFF, x >> 24), u8x2_bf16(y & 0xFF, (y >> 8) & 0xFF),
              u8x2_bf16((y >> 16) & 0xFF, y >> 24));
    }
    // W: fp32 [BN][64] -> bf16 [hi; mid; lo] SW128, rows n, BN + n, 2BN + n
    const uint32_t bst = st + S::A_STG + S::A_BYTES;
    const uint32_t bt = bst + S::B_STG;
#pragma unroll
    for (int j = 0; j < S::BU_PER; ++j) {
      const int u = tid + kProducers * j;
      if (u >= S::BU) break;
      const int r = u >> 3, q = u & 7;
      const float4 a = pipe::lds128(bst + r * 256 + 32 * q);
      const float4 b = pipe::lds128(bst + r * 256 + 32 * q + 16);
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t h[8], m[8], l[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) split3(v[e], h[e], m[e], l[e]);
      sts128u(bt + tc::sw128_off(r, q), pack_hi(h[0], h[1]), pack_hi(h[2], h[3]), pack_hi(h[4], h[5]),
              pack_hi(h[6], h[7]));
      sts128u(bt + tc::sw128_off(BN + r, q), pack_hi(m[0], m[1]), pack_hi(m[2], m[3]), pack_hi(m[4], m[5]),
              pack_hi(m[6], m[7]));
      sts128u(bt + tc::sw128_off(2 * BN + r, q), pack_hi(l[0], l[1]), pack_hi(l[2], l[3]),
              pack_hi(l[4], l[5]), pack_hi(l[6], l[7]));
    }
  };

  if (warp < kMmaWarp) {
    pdl_wait();
#pragma unroll
    for (int c = 0; c < NS - 1; ++c) {
      if (c < nchunks) issue(c, sbase + c * S::STAGE);
      pipe::commit();
    }
  } else {
    tc::tmem_alloc<S::TMEM_COLS>(&tmem_base_sh);
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
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

  if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t id = idesc_bf16(128, 3 * BN);
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % NS;
        tc::mbar_wait(&ready[s], (i / NS) & 1);
        tc::tc_fence_after();
        const uint32_t st = sbase + s * S::STAGE;
        const uint32_t at = st + S::A_STG;
        const uint32_t bt = st + S::A_STG + S::A_BYTES + S::B_STG;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // 4 x K=16 (32 bytes) per 128-byte row
          mma_bf16(tmem, tc::sdesc_sw128(at + kk * 32, 16, 1024), tc::sdesc_sw128(bt + kk * 32, 16, 1024), id,
                   (i | kk) != 0);
        tc::mma_commit(&done[s]);
      }
      tc::mma_commit(&acc_bar);
    }
  } else {
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % NS;
      const uint32_t st = sbase + s * S::STAGE;
      pipe::wait_group<NS - 2>();
      convert(st);
      tc::fence_async_smem();
      mbar_arrive(&ready[s]);
      const int nc = i + NS - 1;
      if (nc < nchunks) {
        const int ps = nc % NS;
        if (i >= 1) tc::mbar_wait(&done[ps], ((i - 1) / NS) & 1);
        issue(nc, sbase + ps * S::STAGE);
      }
      pipe::commit();
    }
    // ---- epilogue: acc = hi + mid + lo ranges, x 1/256, + bias, ReLU
    if (tid < BN) bias_sh[tid] = n0 + tid < N ? __ldg(epi.bias + n0 + tid) : 0.f;
    asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
    if (nchunks > 0) tc::mbar_wait(&acc_bar, 0);
    tc::tc_fence_after();
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const int cbeg = (warp >> 2) * HALF;
    float* stg = reinterpret_cast<float*>(smem);
    constexpr int PR = BN + 4;
    if (cbeg < BN) {
#pragma unroll 1
      for (int c = 0; c < HALF; c += 16) {
        const int c0 = cbeg + c;
        float v[16], w[16], x[16];
        const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        tc::tmem_ld16(trow + c0, v);
        tc::tmem_ld16(trow + BN + c0, w);
        tc::tmem_ld16(trow + 2 * BN + c0, x);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ((v[j] + w[j]) + x[j]) * (1.0f / 256.0f);
        if (csplit) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(stg + r * PR + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 q;
            q.x = relu(v[j] + bias_sh[c0 + j]);
            q.y = relu(v[j + 1] + bias_sh[c0 + j + 1]);
            q.z = relu(v[j + 2] + bias_sh[c0 + j + 2]);
            q.w = relu(v[j + 3] + bias_sh[c0 + j + 3]);
            *reinterpret_cast<float4*>(stg + r * PR + c0 + j) = q;
          }
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
    const int mvalid = min(128, M - m0);
    const int v4 = min(BN, N - n0) / 4;
    if (!csplit) {
      for (int e = tid; e < mvalid * v4; e += kProducers) {
        const int rr = e / v4, q = e - rr * v4;
        *reinterpret_cast<float4*>(epi.out + static_cast<std::size_t>(m0 + rr) * epi.ldo + n0 + 4 * q) =
            *reinterpret_cast<const float4*>(stg + rr * PR + 4 * q);
      }
    }
  }
  // split-K: reduce the partial tiles through DSMEM.  The cluster barriers
  // are .aligned: every warp reaches them converged, outside the role code.
  if (csplit) {
#ifdef GA3C_PROBE_SYNC
    __syncthreads();
#endif
    tc::cluster_sync();
    if (warp < kMmaWarp) {
      constexpr int PR = BN + 4;
      const int mvalid = min(128, M - m0);
      const int v4 = min(BN, N - n0) / 4;
      const int KS = gridDim.y;
      const int rank = static_cast<int>(tc::cluster_rank());
      const int RB = (128 + KS - 1) / KS;
      const int r0 = rank * RB, r1 = min(mvalid, r0 + RB);
      for (int e = tid; e < (r1 - r0) * v4; e += kProducers) {
        const int rr = r0 + e / v4, q = e % v4;
        const uint32_t off = sbase + static_cast<uint32_t>((rr * PR + 4 * q) * 4);
        float4 a = tc::ld_dsmem4(tc::mapa(off, 0));
        for (int k = 1; k < KS; ++k) {
          const float4 b = tc::ld_dsmem4(tc::mapa(off, k));
          a.x += b.x;
          a.y += b.y;
          a.z += b.z;
          a.w += b.w;
        }
        const int cc = 4 * q;
        a.x = relu(a.x + bias_sh[cc]);
        a.y = relu(a.y + bias_sh[cc + 1]);
        a.z = relu(a.z + bias_sh[cc + 2]);
        a.w = relu(a.w + bias_sh[cc + 3]);
        *reinterpret_cast<float4*>(epi.out + static_cast<std::size_t>(m0 + rr) * epi.ldo + n0 + cc) = a;
      }
    }
    tc::cluster_sync();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace bf
}  // namespace ga3c
