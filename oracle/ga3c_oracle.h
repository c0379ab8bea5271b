/*
 * ga3c_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU fp64 restatement of the GA3C hot path of the reference `qac` library
 * (/root/reference/proj), extended with NHWC/OHWI convolution layers that the
 * reference does not have.  It is the checker for the CUDA
 * product in paper_1611_06256_b200/ and nothing else: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product library never links or calls it.
 *
 * Parity pinning:
 *   - MLP specs (n_conv == 0) are checked BITWISE against the reference's own
 *     nnet.cpp / returns.cpp compiled from /root/reference into oracle/_ref
 *     (oracle/Makefile), and against committed golden vectors generated from it
 *     (tests/golden/make_golden.py).
 *   - Conv layers are pinned by the "conv == dense" bridge (a full-size stride-1
 *     kernel must reproduce nnet::affine bit for bit), by the reference's own
 *     finite-difference method (test_nnet.cpp:21-95) and by an independent
 *     torch float64 autograd restatement in tests/.
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef GA3C_ORACLE_H
#define GA3C_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_CONV 4
#define ORC_MAX_HIDDEN 4

/* Same memory layout as ga3c_net_spec in include/ga3c.h.
 * Reference NetworkSpec (nnet.hpp:14-18) {input_dim, hidden_dims, n_actions}
 * is the special case in_h = in_w = 1, in_c = input_dim, n_conv = 0. */
typedef struct orc_spec {
  int in_h, in_w, in_c;
  int n_conv;
  int conv_out[ORC_MAX_CONV];
  int conv_k[ORC_MAX_CONV];
  int conv_stride[ORC_MAX_CONV];
  int n_hidden;
  int hidden[ORC_MAX_HIDDEN];
  int n_actions;
} orc_spec;

/* Hyperparams, nnet.hpp:20-31 (same layout as ga3c_hyper). */
typedef struct orc_hyper {
  double gamma;
  int t_max;
  double beta;
  double eps_log;
  double eta;
  double alpha;
  double eps_rms;
  double value_loss_weight;
  double grad_clip_norm;
  int clip_rewards;
} orc_hyper;

enum { ORC_OK = 0, ORC_INVALID = 1 };

/* ---- util.hpp:19-63 ---- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t base, const uint64_t* salts, int n_salts);
/* n draws of next_uniform() from std::mt19937_64(seed) (util.hpp:41-43) */
void orc_uniforms(uint64_t seed, double* out, size_t n);
/* raw mt19937_64 outputs */
void orc_mt64(uint64_t seed, uint64_t* out, size_t n);
int orc_sample_index(const double* probs, int n, double u);
int orc_argmax_index(const double* values, int n);

/* ---- nnet ---- */
int orc_validate_spec(const orc_spec* s);
int orc_validate_hyper(const orc_hyper* hp);
size_t orc_param_count(const orc_spec* s); /* 0 if invalid */
size_t orc_input_dim(const orc_spec* s);
int orc_init_model(const orc_spec* s, uint64_t seed, double* theta);
/* states: B x input_dim doubles (NHWC flatten). pi: B x n_actions, v: B. */
int orc_forward(const orc_spec* s, const double* theta, const double* states, int B, double* pi,
                double* v);
double orc_policy_entropy(const double* policy, int n, double eps_log);
/* dtheta: P doubles (overwritten). scalars: {policy_loss, value_loss, entropy}. */
int orc_loss_and_gradients(const orc_spec* s, const orc_hyper* hp, const double* theta,
                           const double* states, const int* actions, const double* returns, int B,
                           double* dtheta, double* scalars);
/* returns 1 if applied, 0 if rejected (non-finite), -1 if invalid */
int orc_rmsprop_update(const orc_hyper* hp, const double* theta, const double* g,
                       const double* dtheta, size_t P, double* theta_out, double* g_out);
/* fp32 restatement of the same update with the exact operation order the
 * CUDA kernel uses (no contraction); used to pin the kernel bitwise. */
int orc_rmsprop_update_f32(float alpha, float one_minus_alpha, float eta, float eps_rms,
                           const float* theta, const float* g, const float* dtheta, size_t P,
                           float* theta_out, float* g_out);

/* ---- returns.cpp:8-26 ---- */
int orc_compute_returns(const double* rewards, int n, int terminal, double bootstrap, double gamma,
                        double* out);

/* ---- CPU baseline: one independent worker per thread, each running
 * forward (mode 0) or loss_and_gradients (mode 1) on its own copy of the
 * batch for `seconds`.  Returns items/s summed over threads. ---- */
double orc_throughput(const orc_spec* s, const orc_hyper* hp, const double* theta,
                      const double* states, const int* actions, const double* returns, int B,
                      int mode, int n_threads, double seconds, long* items_done);

#ifdef __cplusplus
}
#endif
#endif
