// tc_pipe.cuh -- cp.async staging helpers for the tcgen05 pipelines
// (kind::tf32, 3xTF32): ring-depth rules, cp.async wrappers, u8 widening and
// the K-major tile loaders used by tc_ws.cuh.
//
// The tensor core reads an fp32 operand by TRUNCATING it to tf32 (measured on
// B200, tools/tc_probe.cu).  So the raw fp32 bytes, copied global->shared
// with cp.async straight into the 128B-swizzled canonical layout, already
// are the "hi" operand; only lo = x - trunc_tf32(x) is computed (smem->smem).
// u8 frames are staged raw and widened to f32 (exact, no lo).
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

// ----------------------------------------------------------- MN-major tiles
// 32 k-rows (pixels) x E MN elements in the SWIZZLE_128B_BASE32B layout
// (tc_wgrad.cuh detail::mn_off): MN atoms of 32 at 512 B (LBO), 4-row k
// groups at SBO = (E/32)*512.
}  // namespace pipe
}  // namespace ga3c
