// kernels.cu -- the non-GEMM kernels of the GA3C hot path (sm_100a).
//
//   heads_forward_kernel   FC finalize (split-K reduce + bias + ReLU) fused with
//                          the policy/value heads and the max-subtracted softmax
//                          (nnet.cpp:96-117)
//   heads_loss_kernel      the same heads fused with the per-sample A3C loss
//                          terms, dL/dpi, softmax Jacobian, dV, and the heads'
//                          input gradient with the ReLU gate (nnet.cpp:229-270)
//   heads_wgrad_kernel     the heads' weight gradient dhead^T [h | 1] and the
//                          loss diagnostics' batch sums (nnet.cpp:233-262)
//   conv_dgrad_kernel      gather-form col2im of a VALID conv, gated by the
//                          previous layer's activation (nnet.cpp:267-278)
//   splitk_* kernels       fixed-order split-K reductions (deterministic)
//   scalars / clip         loss diagnostics (wide-heads fallback) and the
//                          optional global-norm clip (nnet.cpp:233-235, 281-289)
//   rmsprop_kernel         fused vectorised non-centred RMSProp with the
//                          non-finite reject gate (nnet.cpp:293-312)
//   returns_kernel         n-step returns, fp64 without contraction (returns.cpp:21-24)
//   sample_kernel          inverse-CDF action sampling (util.hpp:46-54)
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "pdl.cuh"

namespace ga3c {

#ifdef GA3C_HTRACE
__device__ unsigned long long g_htrace[32];
#define HTRACE(i)                                                       \
  do {                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                          \
      unsigned long long t_;                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));             \
      g_htrace[i] = t_;                                                 \
    }                                                                   \
  } while (0)
#else
#define HTRACE(i) \
  do {            \
  } while (0)
#endif

namespace {

constexpr int kMaxA = 64;  // n_actions limit (validated by the engine)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace

// ------------------------------------------------------------------ heads
// Shared pieces of the two heads kernels (one CTA per sample):
//   heads_h       h = ReLU(sum_s part[s][b][:] + bias) when the last trunk
//                 layer is an FC whose split-K partials are handed over
//                 (part != null; eight interleaved chains combined in a fixed
//                 order: independent loads in flight, reproducible result),
//                 else h is read from h_in;
//   heads_logits  logits / value in fp32 (fixed-order block reduction);
//   softmax       max-subtracted softmax in fp64, one lane per action for
//                 exp(), the normaliser summed in action order (nnet.cpp:110-117).
__device__ __forceinline__ void heads_h(const float* __restrict__ part, int n_split,
                                        const float* __restrict__ fc_bias, float* __restrict__ h_io, int B,
                                        int D, int b, float* h) {
  float* hrow = h_io + static_cast<std::size_t>(b) * D;
  for (int o = threadIdx.x; o < D; o += blockDim.x) {
    float v;
    if (part) {
      // 16 loads in flight per round; split k accumulates into chain k % 8
      float c[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const std::size_t stride = static_cast<std::size_t>(B) * D;
      const float* pp = part + static_cast<std::size_t>(b) * D + o;
      for (int k = 0; k < n_split; k += 16) {
        float t[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = k + u < n_split ? pp[(k + u) * stride] : 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u) c[u & 7] += t[u];
      }
      const float s = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]));
      v = s + fc_bias[o];
      v = v < 0.0f ? 0.0f : v;
      hrow[o] = v;
    } else {
      v = hrow[o];
    }
    h[o] = v;
  }
}

// Head weights [A][D] policy rows then the value row -> smem (4-byte
// cp.async: the offsets carry no alignment guarantee); completes with
// heads_w_wait().  Issued first so it overlaps the partial reduction.
__device__ __forceinline__ void heads_w_issue(const float* __restrict__ theta, std::size_t wp_off,
                                              std::size_t wv_off, int A, int D, float* w) {
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(w));
  const int n = (A + 1) * D;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float* src = i < A * D ? theta + wp_off + i : theta + wv_off + (i - A * D);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sb + 4u * i), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void heads_w_wait() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
}

// Returns (in warp 0, all lanes) nothing; writes logit_sh[0..A) (as double)
// and *val_sh = value.  Must be called by the whole CTA.
// bias_j: lane j of warp 0 holds the bias of output j (j <= A), prefetched
// at kernel start.  All (A+1) dot products run in one pass over h with
// independent accumulators and interleaved warp reductions.
__device__ __forceinline__ void heads_logits(int A, int D, const float* wsm, const float* h, float bias_j,
                                             float* red, double* logit_sh, float* val_sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (A + 1 <= 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int o = tid; o < D; o += blockDim.x) {
      const float x = h[o];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j <= A) acc[j] = fmaf(wsm[static_cast<std::size_t>(j) * D + o], x, acc[j]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j <= A) red[warp * (A + 1) + j] = acc[j];
    }
  } else {
    for (int j = 0; j <= A; ++j) {
      const float* w = wsm + static_cast<std::size_t>(j) * D;
      float sacc = 0.0f;
      for (int o = tid; o < D; o += blockDim.x) sacc = fmaf(w[o], h[o], sacc);
      sacc = warp_sum(sacc);
      if (lane == 0) red[warp * (A + 1) + j] = sacc;
    }
  }
  __syncthreads();
  if (warp == 0) {
    for (int j = lane; j <= A; j += 32) {
      float sacc = 0.0f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sacc += red[w * (A + 1) + j];
      const float z = sacc + bias_j;
      if (j < A)
        logit_sh[j] = z;
      else
        *val_sh = z;
    }
  }
  __syncthreads();
}

// p[0..A) = softmax(logit_sh) in fp64; whole CTA calls, warp 0 computes.
__device__ __forceinline__ void softmax64(const double* logit_sh, int A, double* e_sh, double* p_sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    double m = logit_sh[0];
    for (int j = 1; j < A; ++j)
      if (m < logit_sh[j]) m = logit_sh[j];
    for (int j = lane; j < A; j += 32) e_sh[j] = exp(logit_sh[j] - m);
    __syncwarp();
    if (lane == 0) {
      double z = 0.0;
      for (int j = 0; j < A; ++j) z += e_sh[j];
      e_sh[A] = z;
    }
    __syncwarp();
    const double z = e_sh[A];
    for (int j = lane; j < A; j += 32) p_sh[j] = e_sh[j] / z;
  }
  __syncthreads();
}

// Predictor forward: FC finalize + heads + softmax.  pi64 (internal, for the
// sampler) and pi32 (API output), V in fp32 and fp64.
__global__ void __launch_bounds__(256)
heads_forward_kernel(const float* __restrict__ part, int n_split, const float* __restrict__ fc_bias,
                     float* __restrict__ h_io, int B, int D, const float* __restrict__ theta,
                     std::size_t wp_off, std::size_t bp_off, std::size_t wv_off, std::size_t bv_off,
                     int A, float* __restrict__ pi32, double* __restrict__ pi64,
                     float* __restrict__ v_out, double* __restrict__ v64_out) {
  pdl_enter();
  extern __shared__ float sm[];
  float* h = sm;                 // D
  float* red = sm + D;           // [8 warps][A+1]
  float* wsm = red + 8 * (A + 1);  // [A+1][D] head weights
  __shared__ double logit_sh[kMaxA], e_sh[kMaxA + 1], p_sh[kMaxA];
  __shared__ float val_sh;
  const int b = blockIdx.x;
  heads_w_issue(theta, wp_off, wv_off, A, D, wsm);
  const int lane = threadIdx.x & 31;
  const float bias_j = threadIdx.x < 32 && lane <= A ? theta[lane < A ? bp_off + lane : bv_off] : 0.f;
  heads_h(part, n_split, fc_bias, h_io, B, D, b, h);
  heads_w_wait();
  heads_logits(A, D, wsm, h, bias_j, red, logit_sh, &val_sh);
  softmax64(logit_sh, A, e_sh, p_sh);
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    pi64[static_cast<std::size_t>(b) * A + j] = p_sh[j];
    pi32[static_cast<std::size_t>(b) * A + j] = static_cast<float>(p_sh[j]);
  }
  if (threadIdx.x == 0) {
    v_out[b] = val_sh;
    v64_out[b] = val_sh;
  }
}

// Trainer: the forward's heads fused with the loss and the heads' backward,
// one CTA per sample (nnet.cpp:229-270):
//   fp64 loss algebra from pi and V (advantage constant in the policy term),
//   dL/dlogits through the softmax Jacobian, dV, then
//   dh = W_p^T dlogits + W_v dV in fp32 gated by h <= 0 (written row-major
//   for the conv path and transposed for the FC input-gradient GEMM), the
//   per-sample head gradients dhead[b] for the heads' weight gradient, and
//   the per-sample loss diagnostics, whose fixed-order batch sum the last
//   CTA to finish computes (ticket counter, no float atomics).
__global__ void __launch_bounds__(256)
heads_loss_kernel(const float* __restrict__ part, int n_split, const float* __restrict__ fc_bias,
                  float* __restrict__ h_io, int B, int D, const float* __restrict__ theta,
                  std::size_t wp_off, std::size_t bp_off, std::size_t wv_off, std::size_t bv_off, int A,
                  const int32_t* __restrict__ actions, const double* __restrict__ rets, double beta,
                  double eps, double c_v, double* __restrict__ pi64, float* __restrict__ v_out,
                  float* __restrict__ dhead, float* __restrict__ dh, float* __restrict__ dhT, int ldT,
                  double* __restrict__ scal, int* __restrict__ flag) {
  pdl_enter();
  // every dtheta writer of this step runs after this kernel: reset the
  // non-finite flag here (stream order) instead of a separate memset node
  if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 0;
  HTRACE(0);
  extern __shared__ float sm[];
  float* h = sm;
  float* red = sm + D;
  float* wsm = red + 8 * (A + 1);  // [A+1][D] head weights
  __shared__ double logit_sh[kMaxA], e_sh[kMaxA + 1], p_sh[kMaxA], lg_sh[kMaxA], dp_sh[kMaxA];
  __shared__ float val_sh, g_sh[kMaxA + 1];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  heads_w_issue(theta, wp_off, wv_off, A, D, wsm);
  HTRACE(1);
  // small per-sample inputs, fetched now so their latency hides under the
  // partial reduction
  const float bias_j = tid < 32 && lane <= A ? theta[lane < A ? bp_off + lane : bv_off] : 0.f;
  const int a = tid < 32 ? actions[b] : 0;
  const double ret_b = tid < 32 ? rets[b] : 0.0;
  heads_h(part, n_split, fc_bias, h_io, B, D, b, h);
  HTRACE(2);
  heads_w_wait();
  HTRACE(3);
  heads_logits(A, D, wsm, h, bias_j, red, logit_sh, &val_sh);
  HTRACE(4);
  softmax64(logit_sh, A, e_sh, p_sh);
  HTRACE(5);
  if (tid < 32) {
    // an action outside [0, A) (the reference throws, nnet.cpp:214-216) makes
    // the sample's advantage NaN, so every gradient it touches is non-finite
    // and the step is rejected by the flag the gradient writers raise
    const bool bad_a = static_cast<unsigned>(a) >= static_cast<unsigned>(A);
    const double adv = bad_a ? __longlong_as_double(0x7ff8000000000000ULL) : ret_b - static_cast<double>(val_sh);
    const int ac = bad_a ? 0 : a;
    for (int k = lane; k < A; k += 32) {
      const double p = p_sh[k];
      pi64[static_cast<std::size_t>(b) * A + k] = p;
      lg_sh[k] = log(p + eps);  // eps > 0 (validated)
      double d = beta * (lg_sh[k] + p / (p + eps));
      if (k == a) d += -adv / (p + eps);
      dp_sh[k] = d;
    }
    __syncwarp();
    if (lane == 0) {
      v_out[b] = val_sh;
      double H = 0.0, dot = 0.0;
      for (int k = 0; k < A; ++k) H -= p_sh[k] * lg_sh[k];
      for (int k = 0; k < A; ++k) dot += dp_sh[k] * p_sh[k];
      scal[3 * b + 0] = -lg_sh[ac] * adv - beta * H;
      scal[3 * b + 1] = adv * adv;
      scal[3 * b + 2] = H;
      e_sh[0] = dot;
      const float dvv = static_cast<float>(-2.0 * c_v * adv);
      g_sh[A] = dvv;
      dhead[static_cast<std::size_t>(b) * (A + 1) + A] = dvv;
    }
    __syncwarp();
    const double dot = e_sh[0];
    for (int j = lane; j < A; j += 32) {
      const float g = static_cast<float>(p_sh[j] * (dp_sh[j] - dot));
      g_sh[j] = g;
      dhead[static_cast<std::size_t>(b) * (A + 1) + j] = g;
    }
  }
  __syncthreads();
  HTRACE(6);
  if (dh) {
    float* drow = dh + static_cast<std::size_t>(b) * D;
    for (int o = tid; o < D; o += blockDim.x) {
      float s = 0.0f;
      for (int j = 0; j < A; ++j) s = fmaf(g_sh[j], wsm[static_cast<std::size_t>(j) * D + o], s);
      s = fmaf(g_sh[A], wsm[static_cast<std::size_t>(A) * D + o], s);
      const float g = h[o] <= 0.0f ? 0.0f : s;
      drow[o] = g;
      if (dhT) dhT[static_cast<std::size_t>(o) * ldT + b] = g;
    }
  }
  HTRACE(7);
  HTRACE(9);
}

// Fixed-order batch sums of the per-sample diagnostics (nnet.cpp:233-235)
// (heads too wide for final_grad_kernel's heads blocks).
__global__ void scalars_kernel(const double* __restrict__ scal, int B, double* __restrict__ out) {
  pdl_enter();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int b = 0; b < B; ++b) s += scal[3 * b + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// ------------------------------------------------------------ conv dgrad
// din[b][y][x][ci] = gate > 0 ? sum_{ky,kx,co} dout[b][oy][ox][co] W[co][ky][kx][ci] : 0
// over the (ky, kx) with y = oy*s + ky, x = ox*s + kx inside the output.
__global__ void __launch_bounds__(256)
conv_dgrad_kernel(const float* __restrict__ dout, const float* __restrict__ W,
                  const float* __restrict__ gate, float* __restrict__ din, int B, int ih, int iw,
                  int cin, int oh, int ow, int cout, int k, int s) {
  pdl_enter();
  const std::size_t total = static_cast<std::size_t>(B) * ih * iw * cin;
  const std::size_t idx = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  if (gate[idx] <= 0.0f) {
    din[idx] = 0.0f;
    return;
  }
  const int ci = static_cast<int>(idx % cin);
  std::size_t r = idx / cin;
  const int x = static_cast<int>(r % iw);
  r /= iw;
  const int y = static_cast<int>(r % ih);
  const int b = static_cast<int>(r / ih);
  float acc = 0.0f;
  for (int ky = y % s; ky < k; ky += s) {
    const int oy = (y - ky) / s;
    if (oy < 0 || oy >= oh) continue;
    for (int kx = x % s; kx < k; kx += s) {
      const int ox = (x - kx) / s;
      if (ox < 0 || ox >= ow) continue;
      const float* g = dout + ((static_cast<std::size_t>(b) * oh + oy) * ow + ox) * cout;
      const float* w = W + (static_cast<std::size_t>(ky) * k + kx) * cin + ci;
      const std::size_t wstride = static_cast<std::size_t>(k) * k * cin;
      for (int co = 0; co < cout; ++co) acc = fmaf(__ldg(g + co), __ldg(w + co * wstride), acc);
    }
  }
  din[idx] = acc;
}

// Input gradient of a VALID conv.  A CTA covers 64 input pixels x 16 input
// channels (blockIdx.y = channel chunk); each thread owns one pixel x 4
// channels.  The W[co][ky][kx][ci0:+16] slice is staged in shared memory
// once per CTA and dout rows are read as float4.  Same math and gating as
// conv_dgrad_kernel (nnet.cpp:267-278), with ~30x fewer loads.
__global__ void __launch_bounds__(256)
conv_dgrad16_kernel(const float* __restrict__ dout, const float* __restrict__ W,
                    const float* __restrict__ gate, float* __restrict__ din, int B, int ih, int iw,
                    int cin, int oh, int ow, int cout, int k, int s) {
  pdl_enter();
  extern __shared__ float4 wsh4[];  // [cout][k][k][4 groups] float4
  const int ci0 = blockIdx.y * 16;
  const int kk2 = k * k;
  for (int i = threadIdx.x; i < cout * kk2 * 4; i += blockDim.x) {
    const int q = i & 3, r = i >> 2;  // r = co*kk2 + (ky*k + kx)
    wsh4[i] = *reinterpret_cast<const float4*>(W + static_cast<std::size_t>(r) * cin + ci0 + 4 * q);
  }
  __syncthreads();
  const int grp = threadIdx.x & 3;
  const int pix = blockIdx.x * 64 + (threadIdx.x >> 2);
  if (pix >= B * ih * iw) return;
  const int x = pix % iw;
  const int y = (pix / iw) % ih;
  const int b = pix / (iw * ih);
  const std::size_t base = static_cast<std::size_t>(pix) * cin + ci0 + 4 * grp;
  const float4 gt = *reinterpret_cast<const float4*>(gate + base);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gt.x > 0.f || gt.y > 0.f || gt.z > 0.f || gt.w > 0.f) {
    for (int ky = y % s; ky < k; ky += s) {
      const int oy = (y - ky) / s;
      if (y < ky || oy >= oh) continue;
      for (int kx = x % s; kx < k; kx += s) {
        const int ox = (x - kx) / s;
        if (x < kx || ox >= ow) continue;
        const float4* g4 =
            reinterpret_cast<const float4*>(dout + ((static_cast<std::size_t>(b) * oh + oy) * ow + ox) * cout);
        const float4* w4 = wsh4 + (ky * k + kx) * 4 + grp;
        for (int c4 = 0; c4 < cout / 4; ++c4) {
          const float4 d = __ldg(g4 + c4);
          const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 w = w4[(4 * c4 + c) * kk2 * 4];
            acc.x = fmaf(dv[c], w.x, acc.x);
            acc.y = fmaf(dv[c], w.y, acc.y);
            acc.z = fmaf(dv[c], w.z, acc.z);
            acc.w = fmaf(dv[c], w.w, acc.w);
          }
        }
      }
    }
  }
  float4 o;
  o.x = gt.x <= 0.f ? 0.f : acc.x;
  o.y = gt.y <= 0.f ? 0.f : acc.y;
  o.z = gt.z <= 0.f ? 0.f : acc.z;
  o.w = gt.w <= 0.f ? 0.f : acc.w;
  *reinterpret_cast<float4*>(din + base) = o;
}

// Same contraction with the shape known at compile time (the GA3C stacks:
// k = 4, s = 2, COUT = 32 / 64): the weight slice arrives by cp.async, the
// gate load overlaps it, and each tap's COUT/4 dout vectors are issued back
// to back, so a thread waits for one round trip per tap instead of one per
// vector.  Result identical to conv_dgrad16_kernel (same summation order).
template <int COUT, int K, int S>
__device__ __forceinline__ void conv_dgrad_t_body(const float* __restrict__ dout, const float* __restrict__ W,
                                                  const float* __restrict__ gate, float* __restrict__ din, int B,
                                                  int ih, int iw, int cin, int oh, int ow) {
  constexpr int KK2 = K * K;
  constexpr int NV = COUT * KK2 * 4;  // float4 slots of the [co][ky][kx][16 ci] slice
  extern __shared__ float4 wsh4[];
  pdl_enter();
  const int ci0 = blockIdx.y * 16;
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(wsh4));
#pragma unroll
  for (int j = 0; j < (NV + 255) / 256; ++j) {
    const int i = threadIdx.x + 256 * j;
    if (i < NV) {
      const int q = i & 3, r = i >> 2;
      const float* src = W + static_cast<std::size_t>(r) * cin + ci0 + 4 * q;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + 16u * i), "l"(src) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int grp = threadIdx.x & 3;
  const int pix = blockIdx.x * 64 + (threadIdx.x >> 2);
  const bool live = pix < B * ih * iw;
  const int x = live ? pix % iw : 0;
  const int y = live ? (pix / iw) % ih : 0;
  const int b = live ? pix / (iw * ih) : 0;
  const std::size_t base = static_cast<std::size_t>(live ? pix : 0) * cin + ci0 + 4 * grp;
  const float4 gt = live ? *reinterpret_cast<const float4*>(gate + base) : make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (!live) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gt.x > 0.f || gt.y > 0.f || gt.z > 0.f || gt.w > 0.f) {
#pragma unroll
    for (int ty = 0; ty < K / S; ++ty) {
      const int ky = y % S + S * ty;
      const int oy = (y - ky) / S;
      if (y < ky || oy >= oh) continue;
#pragma unroll
      for (int tx = 0; tx < K / S; ++tx) {
        const int kx = x % S + S * tx;
        const int ox = (x - kx) / S;
        if (x < kx || ox >= ow) continue;
        const float4* g4 =
            reinterpret_cast<const float4*>(dout + ((static_cast<std::size_t>(b) * oh + oy) * ow + ox) * COUT);
        float4 d[COUT / 4];
#pragma unroll
        for (int c4 = 0; c4 < COUT / 4; ++c4) d[c4] = __ldg(g4 + c4);
        const float4* w4 = wsh4 + (ky * K + kx) * 4 + grp;
#pragma unroll
        for (int c4 = 0; c4 < COUT / 4; ++c4) {
          const float dv[4] = {d[c4].x, d[c4].y, d[c4].z, d[c4].w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 w = w4[(4 * c4 + c) * KK2 * 4];
            acc.x = fmaf(dv[c], w.x, acc.x);
            acc.y = fmaf(dv[c], w.y, acc.y);
            acc.z = fmaf(dv[c], w.z, acc.z);
            acc.w = fmaf(dv[c], w.w, acc.w);
          }
        }
      }
    }
  }
  float4 o;
  o.x = gt.x <= 0.f ? 0.f : acc.x;
  o.y = gt.y <= 0.f ? 0.f : acc.y;
  o.z = gt.z <= 0.f ? 0.f : acc.z;
  o.w = gt.w <= 0.f ? 0.f : acc.w;
  *reinterpret_cast<float4*>(din + base) = o;
}

__global__ void __launch_bounds__(256)
conv_dgrad_32x4s2_kernel(const float* __restrict__ dout, const float* __restrict__ W,
                         const float* __restrict__ gate, float* __restrict__ din, int B, int ih, int iw,
                         int cin, int oh, int ow) {
  conv_dgrad_t_body<32, 4, 2>(dout, W, gate, din, B, ih, iw, cin, oh, ow);
}

__global__ void __launch_bounds__(256)
conv_dgrad_64x4s2_kernel(const float* __restrict__ dout, const float* __restrict__ W,
                         const float* __restrict__ gate, float* __restrict__ din, int B, int ih, int iw,
                         int cin, int oh, int ow) {
  conv_dgrad_t_body<64, 4, 2>(dout, W, gate, din, B, ih, iw, cin, oh, ow);
}

// ------------------------------------------------------- split-K reductions
__global__ void splitk_bias_relu_kernel(const float* __restrict__ part, int n_split, int M, int N,
                                        const float* __restrict__ bias, float* __restrict__ out) {
  pdl_enter();
  const std::size_t total = static_cast<std::size_t>(M) * N;
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  float s = 0.0f;
  for (int k = 0; k < n_split; ++k) s += part[k * total + i];
  const float v = s + bias[i % N];
  out[i] = v < 0.0f ? 0.0f : v;
}

__global__ void splitk_grad_kernel(const float* __restrict__ part, int n_split, int M, int N,
                                   GradMap g) {
  pdl_enter();
  const std::size_t total = static_cast<std::size_t>(M) * N;
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  float s = 0.0f;
  for (int k = 0; k < n_split; ++k) s += part[k * total + i];
  g.store(static_cast<int>(i / N), static_cast<int>(i % N), s);
}

// Many splits: 256 threads = 32 outputs x 8 interleaved sub-sums (split q,
// q+8, ...) combined in sub-sum order -- a fixed reduction tree, so results
// are reproducible run to run.
__global__ void __launch_bounds__(256)
splitk_grad8_kernel(const float* __restrict__ part, int n_split, int M, int N, GradMap g) {
  pdl_enter();
  __shared__ float red[8][33];
  const std::size_t total = static_cast<std::size_t>(M) * N;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * 32 + lane;
  float s = 0.0f;
  if (i < total)
    for (int k = q; k < n_split; k += 8) s += part[k * total + i];
  red[q][lane] = s;
  __syncthreads();
  if (q == 0 && i < total) {
    float t = red[0][lane];
#pragma unroll
    for (int r = 1; r < 8; ++r) t += red[r][lane];
    g.store(static_cast<int>(i / N), static_cast<int>(i % N), t);
  }
}

// Tensor-core weight-gradient partials: weights [split][cout][Kw] (16-byte
// aligned rows) followed by the bias sums [split][cout].  Output element i of
// the virtual [cout][Kw+1] matrix (bias in the last column).
// Element (co, kk) of split k sits at base + k * stride (weights, then the
// bias block).  32-bit index math (cout * (Kw + 1) < 2^31, checked by the
// host), done before the PDL wait so it overlaps the producer's tail.
struct SplitCol {
  std::size_t base, stride;
};
__device__ __forceinline__ SplitCol split_col(int n_split, int cout, int Kw, int co, int kk) {
  if (kk < Kw)
    return {static_cast<std::size_t>(co) * Kw + kk, static_cast<std::size_t>(cout) * Kw};
  return {static_cast<std::size_t>(n_split) * cout * Kw + co, static_cast<std::size_t>(cout)};
}

__global__ void splitk_wgrad_kernel(const float* __restrict__ part, int n_split, int cout, int Kw,
                                    GradMap g) {
  const unsigned N = static_cast<unsigned>(Kw) + 1u;
  const unsigned total = static_cast<unsigned>(cout) * N;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  const int co = static_cast<int>(i / N), kk = static_cast<int>(i - (i / N) * N);
  const SplitCol c = split_col(n_split, cout, Kw, co, kk);
  pdl_enter();
  if (i >= total) return;
  float s = 0.0f;
#pragma unroll 4
  for (int k = 0; k < n_split; ++k) s += part[c.base + k * c.stride];
  g.store(co, kk, s);
}

__global__ void __launch_bounds__(256)
splitk_wgrad8_kernel(const float* __restrict__ part, int n_split, int cout, int Kw, GradMap g) {
  __shared__ float red[8][33];
  const unsigned N = static_cast<unsigned>(Kw) + 1u;
  const unsigned total = static_cast<unsigned>(cout) * N;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const unsigned i = blockIdx.x * 32u + lane;
  const int co = static_cast<int>(i / N), kk = static_cast<int>(i - (i / N) * N);
  const SplitCol c = split_col(n_split, cout, Kw, co, kk);
  pdl_enter();
  float s = 0.0f;
  if (i < total) {
#pragma unroll 4
    for (int k = q; k < n_split; k += 8) s += part[c.base + k * c.stride];
  }
  red[q][lane] = s;
  __syncthreads();
  if (q == 0 && i < total) {
    float t = red[0][lane];
#pragma unroll
    for (int r = 1; r < 8; ++r) t += red[r][lane];
    g.store(co, kk, t);
  }
}

// -------------------------------------------------------------- clipping
__global__ void sumsq_kernel(const float* __restrict__ g, std::size_t n, double* __restrict__ part) {
  pdl_enter();
  __shared__ double red[32];
  double s = 0.0;
  for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const double x = g[i];
    s += x * x;
  }
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void clip_scale_kernel(float* __restrict__ g, std::size_t n, const double* __restrict__ part,
                                  int n_part, double clip) {
  pdl_enter();
  __shared__ double scale_sh;
  if (threadIdx.x == 0) {
    double sq = 0.0;
    for (int i = 0; i < n_part; ++i) sq += part[i];
    const double norm = sqrt(sq);
    scale_sh = norm > clip ? clip / norm : 1.0;
  }
  __syncthreads();
  const double scale = scale_sh;
  if (scale == 1.0) return;
  for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    g[i] = static_cast<float>(static_cast<double>(g[i]) * scale);
}

// --------------------------------------------------------------- rmsprop
// g' = alpha*g + ((1-alpha)*d)*d ; theta' = theta - (eta*d)/sqrt(g' + eps)
// One IEEE rounding per operation (explicit _rn intrinsics, no contraction),
// matching orc_rmsprop_update_f32 bit for bit.  20 B/param of HBM traffic.
// If *flag is set (a non-finite gradient component) the step is rejected and
// nothing is written (nnet.cpp:299-301).  Out-of-place or in place.
__device__ __forceinline__ void rms1(float& th, float& g, float d, float alpha, float oma, float eta,
                                     float eps) {
  const float acc = __fadd_rn(__fmul_rn(alpha, g), __fmul_rn(__fmul_rn(oma, d), d));
  g = acc;
  th = __fsub_rn(th, __fdiv_rn(__fmul_rn(eta, d), __fsqrt_rn(__fadd_rn(acc, eps))));
}

__global__ void __launch_bounds__(256)
rmsprop_kernel(const float* __restrict__ th_in, const float* __restrict__ g_in,
               const float* __restrict__ d, float* __restrict__ th_out, float* __restrict__ g_out,
               std::size_t n, const int* __restrict__ flag, unsigned long long* version, float alpha,
               float oma, float eta, float eps) {
  pdl_enter();
  const std::size_t n4 = n / 4;
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  const std::size_t t0 = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const float4* T = reinterpret_cast<const float4*>(th_in);
  const float4* G = reinterpret_cast<const float4*>(g_in);
  const float4* D = reinterpret_cast<const float4*>(d);
  float4* TO = reinterpret_cast<float4*>(th_out);
  float4* GO = reinterpret_cast<float4*>(g_out);
  // The flag load is issued beside the data loads (its value is only needed
  // at the stores), saving one L2 round trip on the update's critical path.
  // Rejected (nnet.cpp:299-301): an out-of-place destination receives the
  // source unchanged, so the slot ring still holds the latest parameters.
  // (asm: a plain load would be made uniform, and its R2UR stalls the warp
  // on the flag before the data loads issue)
  int flag_v;
  asm volatile("ld.global.b32 %0, [%1];" : "=r"(flag_v) : "l"(flag));
  const bool rejected = flag_v != 0;
  const bool copy = th_out != th_in;
  for (std::size_t i = t0; i < n4; i += stride) {
    float4 t = T[i], g = G[i];
    const float4 dd = __ldcs(D + i);
    if (!rejected) {
      rms1(t.x, g.x, dd.x, alpha, oma, eta, eps);
      rms1(t.y, g.y, dd.y, alpha, oma, eta, eps);
      rms1(t.z, g.z, dd.z, alpha, oma, eta, eps);
      rms1(t.w, g.w, dd.w, alpha, oma, eta, eps);
    }
    if (!rejected || copy) {
      TO[i] = t;
      GO[i] = g;
    }
  }
  for (std::size_t i = n4 * 4 + t0; i < n; i += stride) {
    float t = th_in[i], g = g_in[i];
    const float dd = d[i];
    if (!rejected) rms1(t, g, dd, alpha, oma, eta, eps);
    if (!rejected || copy) {
      th_out[i] = t;
      g_out[i] = g;
    }
  }
  if (rejected) return;
  if (version && t0 == 0) *version += 1ull;
}

// ------------------------------------------------- heads weight gradient
__global__ void __launch_bounds__(256) heads_wgrad_kernel(HeadsGrad hg, float* __restrict__ grad,
                                                          int* __restrict__ flag) {
  __shared__ float hs[64][33];  // h[b][c0 + col] for a chunk of 64 samples
  __shared__ float gs[64][9];   // dhead[b][j] when A + 1 <= 9 (else read directly)
  pdl_enter();
  const int tid = threadIdx.x;
  bool bad = false;
  // columns [c0, c0 + 32) of [h | 1] (column D = the bias), rows
  // j = tid / 32 (+ 8, + 16, + 24) <= A
  const int c0 = static_cast<int>(blockIdx.x) * 32;
  if (c0 == 0 && hg.scal) {
    // the loss diagnostics' batch sums in sample order (scalars_kernel's
    // order), staged 255 terms (85 samples) per round
    __shared__ double sc[256];
    double acc_s = 0.0;
    const int n = 3 * hg.B;
    for (int i0 = 0; i0 < n; i0 += 255) {
      const int m = min(255, n - i0);
      __syncthreads();
      if (tid < m) sc[tid] = __ldcg(hg.scal + i0 + tid);
      __syncthreads();
      if (tid < 3)
        for (int i = tid; i < m; i += 3) acc_s += sc[i];
    }
    if (tid < 3) hg.scal_sum[tid] = acc_s;
  }
  const int col = c0 + (tid & 31);
  const int A1 = hg.A + 1;
  constexpr int kRows = 256 / 32;
  const int nj = (A1 + kRows - 1) / kRows;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int b0 = 0; b0 < hg.B; b0 += 64) {
    const int nb = min(64, hg.B - b0);
    __syncthreads();
    for (int i = tid; i < nb * 32; i += blockDim.x) {
      const int bb = i >> 5, cc = c0 + (i & 31);
      hs[bb][i & 31] = cc < hg.D ? __ldcg(hg.h + static_cast<std::size_t>(b0 + bb) * hg.D + cc) : 1.f;
    }
    if (A1 <= 9)
      for (int i = tid; i < nb * A1; i += blockDim.x) {
        const int bb = i / A1, jj = i - bb * A1;
        gs[bb][jj] = __ldcg(hg.dhead + static_cast<std::size_t>(b0 + bb) * A1 + jj);
      }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = tid / 32 + kRows * q;
      if (q >= nj || j >= A1) break;
      float s = acc[q];
      for (int bb = 0; bb < nb; ++bb) {
        const float g = A1 <= 9 ? gs[bb][j] : __ldcg(hg.dhead + static_cast<std::size_t>(b0 + bb) * A1 + j);
        s = fmaf(g, hs[bb][tid & 31], s);
      }
      acc[q] = s;
    }
  }
  if (col <= hg.D) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = tid / 32 + kRows * q;
      if (q >= nj || j >= A1) break;
      const unsigned long long i = j < hg.A ? (col < hg.D ? hg.wp_off + static_cast<unsigned long long>(j) * hg.D + col
                                                          : hg.bp_off + j)
                                            : (col < hg.D ? hg.wv_off + col : hg.bv_off);
      grad[i] = acc[q];
      bad |= !isfinite(acc[q]);
    }
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);
}

// --------------------------------------------------------------- returns
// returns.cpp:21-24: acc = r_i + gamma * acc, two roundings (no FMA), so the
// result is bitwise equal to the reference's x86-64 build.
__global__ void returns_kernel(const double* __restrict__ rewards, const int32_t* __restrict__ off,
                               int n_seg, const uint8_t* __restrict__ terminal,
                               const double* __restrict__ bootstrap, double gamma,
                               double* __restrict__ out) {
  pdl_enter();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  double acc = terminal[s] ? 0.0 : bootstrap[s];
  for (int i = off[s + 1]; i-- > off[s];) {
    acc = __dadd_rn(rewards[i], __dmul_rn(gamma, acc));
    out[i] = acc;
  }
}

// --------------------------------------------------------------- sampling
// util.hpp:46-54 on the fp64 policy (pi64) or the fp32 API output.
__global__ void sample_kernel(const float* __restrict__ pi32, const double* __restrict__ pi64,
                              const double* __restrict__ u, int B, int A, int32_t* __restrict__ act,
                              int act_stride) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double uu = u[b];
  double acc = 0.0;
  int res = A - 1;
  for (int i = 0; i < A; ++i) {
    acc += pi64 ? pi64[static_cast<std::size_t>(b) * A + i]
                : static_cast<double>(pi32[static_cast<std::size_t>(b) * A + i]);
    if (uu < acc) {
      res = i;
      break;
    }
  }
  act[static_cast<std::size_t>(b) * act_stride] = res;
}

__global__ void check_finite_kernel(const float* __restrict__ x, std::size_t n, int* __restrict__ flag) {
  pdl_enter();
  for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    if (!isfinite(x[i])) atomicOr(flag, 1);
}

}  // namespace ga3c
