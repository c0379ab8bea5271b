// kernels.cuh -- declarations of the non-GEMM kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "gemm_simt.cuh"

namespace ga3c {

__global__ void heads_forward_kernel(const float* part, int n_split, const float* fc_bias, float* h_io,
                                     int B, int D, const float* theta, std::size_t wp_off,
                                     std::size_t bp_off, std::size_t wv_off, std::size_t bv_off,
                                     int A, float* pi32, double* pi64, float* v_out,
                                     double* v64_out);

__global__ void heads_loss_kernel(const float* part, int n_split, const float* fc_bias, float* h_io, int B,
                                  int D, const float* theta, std::size_t wp_off, std::size_t bp_off,
                                  std::size_t wv_off, std::size_t bv_off, int A, const int32_t* actions,
                                  const double* rets, double beta, double eps, double c_v, double* pi64,
                                  float* v_out, float* dhead, float* dh, float* dhT, int ldT, double* scal,
                                  int* flag);

// ------------------------------------------- heads weight gradient
// [W_p | b_p | w_v | b_v] (nnet.hpp layout order) = dhead^T [h | 1]
// (nnet.cpp:237-262 summed over the batch, sample order), plus the loss
// diagnostics' batch sums (nnet.cpp:233-235), in one launch on the
// backward DAG's side stream: CTA k takes columns [32k, 32k + 32) of [h | 1]
// for every output row, staging h and dhead through shared memory.
struct HeadsGrad {
  const float* dhead;  // [B][A+1]
  const float* h;      // [B][D]
  int B, A, D;         // A + 1 <= 32
  unsigned long long wp_off, bp_off, wv_off, bv_off;
  const double* scal;  // per-sample loss diagnostics [B][3] (nullable)
  double* scal_sum;    // their batch sums
};

__global__ void heads_wgrad_kernel(HeadsGrad hg, float* grad, int* flag);


__global__ void scalars_kernel(const double* scal, int B, double* out);

__global__ void conv_dgrad_kernel(const float* dout, const float* W, const float* gate, float* din,
                                  int B, int ih, int iw, int cin, int oh, int ow, int cout, int k,
                                  int s);

__global__ void conv_dgrad_32x4s2_kernel(const float* dout, const float* W, const float* gate, float* din, int B,
                                         int ih, int iw, int cin, int oh, int ow);
__global__ void conv_dgrad_64x4s2_kernel(const float* dout, const float* W, const float* gate, float* din, int B,
                                         int ih, int iw, int cin, int oh, int ow);
__global__ void conv_dgrad16_kernel(const float* dout, const float* W, const float* gate, float* din,
                                    int B, int ih, int iw, int cin, int oh, int ow, int cout, int k,
                                    int s);

__global__ void splitk_bias_relu_kernel(const float* part, int n_split, int M, int N,
                                        const float* bias, float* out);
__global__ void splitk_grad_kernel(const float* part, int n_split, int M, int N, GradMap g);
__global__ void splitk_grad8_kernel(const float* part, int n_split, int M, int N, GradMap g);
__global__ void splitk_wgrad_kernel(const float* part, int n_split, int cout, int Kw, GradMap g);
__global__ void splitk_wgrad8_kernel(const float* part, int n_split, int cout, int Kw, GradMap g);

__global__ void sumsq_kernel(const float* g, std::size_t n, double* part);
__global__ void clip_scale_kernel(float* g, std::size_t n, const double* part, int n_part,
                                  double clip);

__global__ void rmsprop_kernel(const float* th_in, const float* g_in, const float* d, float* th_out,
                               float* g_out, std::size_t n, const int* flag,
                               unsigned long long* version, float alpha, float oma, float eta,
                               float eps);

__global__ void returns_kernel(const double* rewards, const int32_t* off, int n_seg,
                               const uint8_t* terminal, const double* bootstrap, double gamma,
                               double* out);

__global__ void sample_kernel(const float* pi32, const double* pi64, const double* u, int B, int A,
                              int32_t* act, int act_stride);

__global__ void check_finite_kernel(const float* x, std::size_t n, int* flag);

}  // namespace ga3c
