/*
 * ga3c_oracle.c -- TEST INFRASTRUCTURE ONLY (see ga3c_oracle.h).
 *
 * fp64 CPU restatement of the reference qac hot path
 * (/root/reference/proj/src/nnet.cpp, returns.cpp, include/qac/util.hpp),
 * extended with VALID NHWC/OHWI convolutions that follow nnet.cpp's
 * conventions: bias-first in-order accumulation (nnet.cpp:47-56), ReLU as
 * std::max(v, 0.0) (nnet.cpp:99), the ReLU gate on post-activation <= 0
 * (nnet.cpp:268-270), layout order W then b per layer (nnet.cpp:29-45) and
 * init order/bounds (nnet.cpp:152-168) with conv fan_in = k*k*Cin.
 *
 * Compile WITHOUT FMA contraction (-ffp-contract=off, no -march=native): the
 * reference's own Release build on baseline x86-64 has no FMA, and the
 * bitwise bridge against oracle/_ref depends on it.
 */
#include "ga3c_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ util */

/* util.hpp:21-26 */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* util.hpp:28-32 */
uint64_t orc_derive_seed(uint64_t base, const uint64_t* salts, int n_salts) {
  uint64_t h = orc_mix64(base);
  for (int i = 0; i < n_salts; ++i) h = orc_mix64(h ^ salts[i]);
  return h;
}

/* std::mt19937_64 (the engine the reference seeds everywhere). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = 312;
}

static uint64_t mt64_next(mt64* m) {
  if (m->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (m->mt[i] & upper) | (m->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t y = m->mt[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* util.hpp:41-43 */
static double next_uniform(mt64* m) { return (double)(mt64_next(m) >> 11) * 0x1.0p-53; }

void orc_uniforms(uint64_t seed, double* out, size_t n) {
  mt64 m;
  mt64_seed(&m, seed);
  for (size_t i = 0; i < n; ++i) out[i] = next_uniform(&m);
}

void orc_mt64(uint64_t seed, uint64_t* out, size_t n) {
  mt64 m;
  mt64_seed(&m, seed);
  for (size_t i = 0; i < n; ++i) out[i] = mt64_next(&m);
}

/* util.hpp:46-54 (the draw itself is the caller's: u is passed in) */
int orc_sample_index(const double* probs, int n, double u) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += probs[i];
    if (u < acc) return i;
  }
  return n - 1;
}

/* util.hpp:57-63 */
int orc_argmax_index(const double* values, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (values[i] > values[best]) best = i;
  return best;
}

/* ---------------------------------------------------------------- layout */

typedef struct {
  size_t w_off, b_off;
  int in, out;                 /* FC: fan-in / fan-out */
  int is_conv;
  int cin, cout, k, stride;    /* conv geometry */
  int ih, iw, oh, ow;
} slice;

typedef struct {
  slice trunk[ORC_MAX_CONV + ORC_MAX_HIDDEN];
  int n_trunk;
  slice policy, value;
  size_t total;
  int in_dim;
} layout;

static int trunk_out_dim(const slice* s) { return s->is_conv ? s->oh * s->ow * s->cout : s->out; }
static int trunk_in_dim(const slice* s) { return s->is_conv ? s->ih * s->iw * s->cin : s->in; }

/* nnet.cpp:123-130 plus conv geometry (VALID: out = (in - k) / s + 1 >= 1) */
int orc_validate_spec(const orc_spec* s) {
  if (s->in_h <= 0 || s->in_w <= 0 || s->in_c <= 0) return ORC_INVALID;
  if (s->n_actions < 2) return ORC_INVALID;
  if (s->n_conv < 0 || s->n_conv > ORC_MAX_CONV) return ORC_INVALID;
  if (s->n_hidden < 0 || s->n_hidden > ORC_MAX_HIDDEN) return ORC_INVALID;
  int h = s->in_h, w = s->in_w;
  for (int i = 0; i < s->n_conv; ++i) {
    if (s->conv_out[i] <= 0 || s->conv_k[i] <= 0 || s->conv_stride[i] <= 0) return ORC_INVALID;
    if (s->conv_k[i] > h || s->conv_k[i] > w) return ORC_INVALID;
    h = (h - s->conv_k[i]) / s->conv_stride[i] + 1;
    w = (w - s->conv_k[i]) / s->conv_stride[i] + 1;
  }
  for (int i = 0; i < s->n_hidden; ++i)
    if (s->hidden[i] <= 0) return ORC_INVALID;
  return ORC_OK;
}

/* nnet.cpp:131-145 */
int orc_validate_hyper(const orc_hyper* hp) {
  if (!(hp->gamma > 0.0) || hp->gamma > 1.0) return ORC_INVALID;
  if (hp->t_max < 1) return ORC_INVALID;
  if (hp->beta < 0.0) return ORC_INVALID;
  if (!(hp->eps_log > 0.0)) return ORC_INVALID;
  if (!(hp->eta > 0.0)) return ORC_INVALID;
  if (!(hp->alpha >= 0.0) || hp->alpha >= 1.0) return ORC_INVALID;
  if (!(hp->eps_rms > 0.0)) return ORC_INVALID;
  if (hp->value_loss_weight < 0.0) return ORC_INVALID;
  if (hp->grad_clip_norm < 0.0) return ORC_INVALID;
  return ORC_OK;
}

/* nnet.cpp:29-45, conv layers first (W [Cout][k][k][Cin] then b). */
static void layout_of(const orc_spec* s, layout* lo) {
  memset(lo, 0, sizeof(*lo));
  size_t off = 0;
  int h = s->in_h, w = s->in_w, c = s->in_c;
  lo->in_dim = h * w * c;
  for (int i = 0; i < s->n_conv; ++i) {
    slice* sl = &lo->trunk[lo->n_trunk++];
    sl->is_conv = 1;
    sl->cin = c;
    sl->cout = s->conv_out[i];
    sl->k = s->conv_k[i];
    sl->stride = s->conv_stride[i];
    sl->ih = h;
    sl->iw = w;
    sl->oh = (h - sl->k) / sl->stride + 1;
    sl->ow = (w - sl->k) / sl->stride + 1;
    sl->in = sl->k * sl->k * c; /* fan-in */
    sl->out = sl->cout;
    sl->w_off = off;
    sl->b_off = off + (size_t)sl->cout * sl->in;
    off = sl->b_off + (size_t)sl->cout;
    h = sl->oh;
    w = sl->ow;
    c = sl->cout;
  }
  int prev = h * w * c;
  for (int i = 0; i < s->n_hidden; ++i) {
    slice* sl = &lo->trunk[lo->n_trunk++];
    sl->in = prev;
    sl->out = s->hidden[i];
    sl->w_off = off;
    sl->b_off = off + (size_t)prev * sl->out;
    off = sl->b_off + (size_t)sl->out;
    prev = sl->out;
  }
  lo->policy.in = prev;
  lo->policy.out = s->n_actions;
  lo->policy.w_off = off;
  lo->policy.b_off = off + (size_t)prev * s->n_actions;
  off = lo->policy.b_off + (size_t)s->n_actions;
  lo->value.in = prev;
  lo->value.out = 1;
  lo->value.w_off = off;
  lo->value.b_off = off + (size_t)prev;
  off = lo->value.b_off + 1;
  lo->total = off;
}

size_t orc_param_count(const orc_spec* s) {
  if (orc_validate_spec(s) != ORC_OK) return 0;
  layout lo;
  layout_of(s, &lo);
  return lo.total;
}

size_t orc_input_dim(const orc_spec* s) { return (size_t)s->in_h * s->in_w * s->in_c; }

/* nnet.cpp:152-168 */
int orc_init_model(const orc_spec* s, uint64_t seed, double* theta) {
  if (orc_validate_spec(s) != ORC_OK) return ORC_INVALID;
  layout lo;
  layout_of(s, &lo);
  memset(theta, 0, lo.total * sizeof(double));
  mt64 rng;
  mt64_seed(&rng, seed);
  slice* all[ORC_MAX_CONV + ORC_MAX_HIDDEN + 2];
  int n = 0;
  for (int i = 0; i < lo.n_trunk; ++i) all[n++] = &lo.trunk[i];
  all[n++] = &lo.policy;
  all[n++] = &lo.value;
  for (int j = 0; j < n; ++j) {
    const slice* sl = all[j];
    const double bound = 1.0 / sqrt((double)sl->in);
    const size_t cnt = (size_t)sl->in * sl->out;
    for (size_t i = 0; i < cnt; ++i) theta[sl->w_off + i] = (next_uniform(&rng) * 2.0 - 1.0) * bound;
  }
  return ORC_OK;
}

/* --------------------------------------------------------------- forward */

/* nnet.cpp:47-56 */
static void affine(const double* theta, const slice* s, const double* x, double* y) {
  for (int o = 0; o < s->out; ++o) {
    double acc = theta[s->b_off + o];
    const double* row = theta + s->w_off + (size_t)o * s->in;
    for (int i = 0; i < s->in; ++i) acc += row[i] * x[i];
    y[o] = acc;
  }
}

/* Convolution restated in affine()'s order: per output (oy, ox, co) the
 * accumulator starts at the bias and adds W[co][ky][kx][ci] * x in
 * (ky, kx, ci) order -- i.e. affine() over the NHWC receptive field. */
static void conv_fwd(const double* theta, const slice* s, const double* x, double* y) {
  for (int oy = 0; oy < s->oh; ++oy)
    for (int ox = 0; ox < s->ow; ++ox)
      for (int co = 0; co < s->cout; ++co) {
        double acc = theta[s->b_off + co];
        const double* row = theta + s->w_off + (size_t)co * s->in;
        int i = 0;
        for (int ky = 0; ky < s->k; ++ky) {
          const double* xr = x + ((size_t)(oy * s->stride + ky) * s->iw + (size_t)ox * s->stride) * s->cin;
          for (int kx = 0; kx < s->k; ++kx)
            for (int ci = 0; ci < s->cin; ++ci, ++i) acc += row[i] * xr[kx * s->cin + ci];
        }
        y[((size_t)oy * s->ow + ox) * s->cout + co] = acc;
      }
}

/* nnet.cpp:58-73 */
static void affine_backward(const double* theta, const slice* s, const double* x, const double* dy,
                            double* dtheta, double* dx /* may be NULL */, int dx_len) {
  if (dx)
    for (int i = 0; i < dx_len; ++i) dx[i] = 0.0;
  for (int o = 0; o < s->out; ++o) {
    const double g = dy[o];
    dtheta[s->b_off + o] += g;
    const size_t row = s->w_off + (size_t)o * s->in;
    const double* w = theta + row;
    double* dw = dtheta + row;
    for (int i = 0; i < s->in; ++i) {
      dw[i] += g * x[i];
      if (dx) dx[i] += g * w[i];
    }
  }
}

/* affine_backward over every output position, in conv_fwd's loop order. */
static void conv_backward(const double* theta, const slice* s, const double* x, const double* dy,
                          double* dtheta, double* dx /* may be NULL */) {
  if (dx) memset(dx, 0, sizeof(double) * (size_t)s->ih * s->iw * s->cin);
  for (int oy = 0; oy < s->oh; ++oy)
    for (int ox = 0; ox < s->ow; ++ox)
      for (int co = 0; co < s->cout; ++co) {
        const double g = dy[((size_t)oy * s->ow + ox) * s->cout + co];
        dtheta[s->b_off + co] += g;
        const size_t row = s->w_off + (size_t)co * s->in;
        const double* w = theta + row;
        double* dw = dtheta + row;
        int i = 0;
        for (int ky = 0; ky < s->k; ++ky) {
          const size_t base = ((size_t)(oy * s->stride + ky) * s->iw + (size_t)ox * s->stride) * s->cin;
          for (int kx = 0; kx < s->k; ++kx)
            for (int ci = 0; ci < s->cin; ++ci, ++i) {
              const size_t xi = base + (size_t)kx * s->cin + ci;
              dw[i] += g * x[xi];
              if (dx) dx[xi] += g * w[i];
            }
        }
      }
}

typedef struct {
  double* hidden[ORC_MAX_CONV + ORC_MAX_HIDDEN]; /* post-ReLU per trunk layer */
  double* logits;
  double* policy;
  double value;
} acts;

static void acts_alloc(const layout* lo, int n_actions, acts* a) {
  for (int i = 0; i < lo->n_trunk; ++i)
    a->hidden[i] = (double*)malloc(sizeof(double) * (size_t)trunk_out_dim(&lo->trunk[i]));
  a->logits = (double*)malloc(sizeof(double) * (size_t)n_actions);
  a->policy = (double*)malloc(sizeof(double) * (size_t)n_actions);
}

static void acts_free(const layout* lo, acts* a) {
  for (int i = 0; i < lo->n_trunk; ++i) free(a->hidden[i]);
  free(a->logits);
  free(a->policy);
}

/* nnet.cpp:91-119 */
static void forward_one(const double* theta, const layout* lo, int n_actions, const double* state,
                        acts* a) {
  const double* x = state;
  for (int li = 0; li < lo->n_trunk; ++li) {
    const slice* s = &lo->trunk[li];
    double* h = a->hidden[li];
    if (s->is_conv)
      conv_fwd(theta, s, x, h);
    else
      affine(theta, s, x, h);
    const int n = trunk_out_dim(s);
    for (int i = 0; i < n; ++i) h[i] = (h[i] < 0.0) ? 0.0 : h[i]; /* std::max(v, 0.0) */
    x = h;
  }
  affine(theta, &lo->policy, x, a->logits);
  double vout;
  affine(theta, &lo->value, x, &vout);
  a->value = vout;
  /* max-subtracted softmax; std::max_element keeps the first maximum */
  double m = a->logits[0];
  for (int i = 1; i < n_actions; ++i)
    if (m < a->logits[i]) m = a->logits[i];
  double z = 0.0;
  for (int i = 0; i < n_actions; ++i) {
    a->policy[i] = exp(a->logits[i] - m);
    z += a->policy[i];
  }
  for (int i = 0; i < n_actions; ++i) a->policy[i] /= z;
}

/* nnet.cpp:75-81 */
static int check_state(const double* st, size_t dim) {
  for (size_t i = 0; i < dim; ++i)
    if (!isfinite(st[i])) return ORC_INVALID;
  return ORC_OK;
}

/* nnet.cpp:174-191 */
int orc_forward(const orc_spec* s, const double* theta, const double* states, int B, double* pi,
                double* v) {
  if (orc_validate_spec(s) != ORC_OK || B < 0) return ORC_INVALID;
  layout lo;
  layout_of(s, &lo);
  const size_t dim = (size_t)lo.in_dim;
  for (int b = 0; b < B; ++b)
    if (check_state(states + (size_t)b * dim, dim) != ORC_OK) return ORC_INVALID;
  acts a;
  acts_alloc(&lo, s->n_actions, &a);
  for (int b = 0; b < B; ++b) {
    forward_one(theta, &lo, s->n_actions, states + (size_t)b * dim, &a);
    memcpy(pi + (size_t)b * s->n_actions, a.policy, sizeof(double) * (size_t)s->n_actions);
    v[b] = a.value;
  }
  acts_free(&lo, &a);
  return ORC_OK;
}

/* nnet.cpp:193-199 */
double orc_policy_entropy(const double* policy, int n, double eps_log) {
  double h = 0.0;
  for (int i = 0; i < n; ++i) {
    const double p = policy[i];
    if (p > 0.0 || eps_log > 0.0) h -= p * log(p + eps_log);
  }
  return h;
}

/* nnet.cpp:201-291 */
int orc_loss_and_gradients(const orc_spec* s, const orc_hyper* hp, const double* theta,
                           const double* states, const int* actions, const double* returns, int B,
                           double* dtheta, double* scalars) {
  if (orc_validate_spec(s) != ORC_OK || orc_validate_hyper(hp) != ORC_OK) return ORC_INVALID;
  if (B <= 0) return ORC_INVALID; /* empty batch */
  layout lo;
  layout_of(s, &lo);
  const size_t dim = (size_t)lo.in_dim;
  const int A = s->n_actions;
  for (int n = 0; n < B; ++n) {
    if (!isfinite(returns[n])) return ORC_INVALID;
    if (check_state(states + (size_t)n * dim, dim) != ORC_OK) return ORC_INVALID;
    if (actions[n] < 0 || actions[n] >= A) return ORC_INVALID;
  }
  memset(dtheta, 0, sizeof(double) * lo.total);
  double policy_loss = 0.0, value_loss = 0.0, entropy = 0.0;
  const double eps = hp->eps_log;

  int max_dim = lo.in_dim;
  for (int i = 0; i < lo.n_trunk; ++i)
    if (trunk_out_dim(&lo.trunk[i]) > max_dim) max_dim = trunk_out_dim(&lo.trunk[i]);
  double* dpol = (double*)malloc(sizeof(double) * (size_t)A);
  double* dlogits = (double*)malloc(sizeof(double) * (size_t)A);
  double* dx = (double*)malloc(sizeof(double) * (size_t)max_dim);
  double* dnext = (double*)malloc(sizeof(double) * (size_t)max_dim);
  acts a;
  acts_alloc(&lo, A, &a);

  for (int n = 0; n < B; ++n) {
    const double* st = states + (size_t)n * dim;
    const double R = returns[n];
    const int act = actions[n];
    forward_one(theta, &lo, A, st, &a);
    const double adv = R - a.value;
    const double pa = a.policy[act];
    const double H = orc_policy_entropy(a.policy, A, eps);
    policy_loss += -log(pa + eps) * adv - hp->beta * H;
    value_loss += adv * adv;
    entropy += H;

    for (int k = 0; k < A; ++k) {
      const double p = a.policy[k];
      dpol[k] = hp->beta * (log(p + eps) + p / (p + eps));
    }
    dpol[act] += -adv / (pa + eps);
    double dot = 0.0;
    for (int k = 0; k < A; ++k) dot += dpol[k] * a.policy[k];
    for (int j = 0; j < A; ++j) dlogits[j] = a.policy[j] * (dpol[j] - dot);
    const double dvalue = -2.0 * hp->value_loss_weight * adv;

    const double* trunk_out = lo.n_trunk ? a.hidden[lo.n_trunk - 1] : st;
    const int tdim = lo.policy.in;
    affine_backward(theta, &lo.policy, trunk_out, dlogits, dtheta, dx, tdim);
    const double dv[1] = {dvalue};
    affine_backward(theta, &lo.value, trunk_out, dv, dtheta, dnext, tdim);
    for (int i = 0; i < tdim; ++i) dx[i] += dnext[i];

    for (int li = lo.n_trunk - 1; li >= 0; --li) {
      const slice* sl = &lo.trunk[li];
      const int od = trunk_out_dim(sl);
      for (int o = 0; o < od; ++o)
        if (a.hidden[li][o] <= 0.0) dx[o] = 0.0;
      const double* x_in = li == 0 ? st : a.hidden[li - 1];
      /* the input layer's dx is dead work in the reference (nnet.cpp:273-277);
       * it cannot change dtheta, so it is skipped here */
      double* dxi = li == 0 ? NULL : dnext;
      if (sl->is_conv)
        conv_backward(theta, sl, x_in, dx, dtheta, dxi);
      else
        affine_backward(theta, sl, x_in, dx, dtheta, dxi, trunk_in_dim(sl));
      if (li > 0) memcpy(dx, dnext, sizeof(double) * (size_t)trunk_in_dim(sl));
    }
  }

  if (hp->grad_clip_norm > 0.0) {
    double sq = 0.0;
    for (size_t i = 0; i < lo.total; ++i) sq += dtheta[i] * dtheta[i];
    const double norm = sqrt(sq);
    if (norm > hp->grad_clip_norm) {
      const double scale = hp->grad_clip_norm / norm;
      for (size_t i = 0; i < lo.total; ++i) dtheta[i] *= scale;
    }
  }
  scalars[0] = policy_loss;
  scalars[1] = value_loss;
  scalars[2] = entropy;
  free(dpol);
  free(dlogits);
  free(dx);
  free(dnext);
  acts_free(&lo, &a);
  return ORC_OK;
}

/* nnet.cpp:293-312 */
int orc_rmsprop_update(const orc_hyper* hp, const double* theta, const double* g,
                       const double* dtheta, size_t P, double* theta_out, double* g_out) {
  if (orc_validate_hyper(hp) != ORC_OK) return -1;
  for (size_t i = 0; i < P; ++i) {
    if (!isfinite(dtheta[i])) {
      memmove(theta_out, theta, sizeof(double) * P);
      memmove(g_out, g, sizeof(double) * P);
      return 0;
    }
  }
  for (size_t i = 0; i < P; ++i) {
    const double d = dtheta[i];
    double acc = g[i];
    acc = hp->alpha * acc + (1.0 - hp->alpha) * d * d;
    g_out[i] = acc;
    theta_out[i] = theta[i] - hp->eta * d / sqrt(acc + hp->eps_rms);
  }
  return 1;
}

/* The same update in fp32 with one rounding per operation, in the order the
 * CUDA kernel evaluates it (paper_1611_06256_b200/csrc/rmsprop.cu). */
int orc_rmsprop_update_f32(float alpha, float one_minus_alpha, float eta, float eps_rms,
                           const float* theta, const float* g, const float* dtheta, size_t P,
                           float* theta_out, float* g_out) {
  for (size_t i = 0; i < P; ++i) {
    if (!isfinite(dtheta[i])) {
      memmove(theta_out, theta, sizeof(float) * P);
      memmove(g_out, g, sizeof(float) * P);
      return 0;
    }
  }
  for (size_t i = 0; i < P; ++i) {
    volatile float d = dtheta[i];
    volatile float t0 = alpha * g[i];
    volatile float t1 = one_minus_alpha * d;
    volatile float t2 = t1 * d;
    volatile float acc = t0 + t2;
    volatile float den = acc + eps_rms;
    volatile float sq = sqrtf(den);
    volatile float num = eta * d;
    volatile float step = num / sq;
    g_out[i] = acc;
    theta_out[i] = theta[i] - step;
  }
  return 1;
}

/* returns.cpp:8-26 */
int orc_compute_returns(const double* rewards, int n, int terminal, double bootstrap, double gamma,
                        double* out) {
  if (n <= 0) return ORC_INVALID;
  if (!(gamma > 0.0) || gamma > 1.0) return ORC_INVALID;
  for (int i = 0; i < n; ++i)
    if (!isfinite(rewards[i])) return ORC_INVALID;
  if (!terminal && !isfinite(bootstrap)) return ORC_INVALID;
  double acc = terminal ? 0.0 : bootstrap;
  for (int i = n; i-- > 0;) {
    acc = rewards[i] + gamma * acc;
    out[i] = acc;
  }
  return ORC_OK;
}

/* ------------------------------------------------------ CPU throughput */

typedef struct {
  const orc_spec* s;
  const orc_hyper* hp;
  const double* theta;
  const double* states;
  const int* actions;
  const double* returns;
  int B, mode;
  double seconds;
  long items;
  size_t P;
} worker_arg;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* worker(void* p) {
  worker_arg* w = (worker_arg*)p;
  const int A = w->s->n_actions;
  double* pi = (double*)malloc(sizeof(double) * (size_t)w->B * A);
  double* v = (double*)malloc(sizeof(double) * (size_t)w->B);
  double* dth = (double*)malloc(sizeof(double) * w->P);
  double sc[3];
  const double t0 = now_s();
  long items = 0;
  do {
    if (w->mode == 0)
      orc_forward(w->s, w->theta, w->states, w->B, pi, v);
    else
      orc_loss_and_gradients(w->s, w->hp, w->theta, w->states, w->actions, w->returns, w->B, dth, sc);
    items += w->B;
  } while (now_s() - t0 < w->seconds);
  w->items = items;
  free(pi);
  free(v);
  free(dth);
  return NULL;
}

double orc_throughput(const orc_spec* s, const orc_hyper* hp, const double* theta,
                      const double* states, const int* actions, const double* returns, int B,
                      int mode, int n_threads, double seconds, long* items_done) {
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  worker_arg* args = (worker_arg*)malloc(sizeof(worker_arg) * (size_t)n_threads);
  const size_t P = orc_param_count(s);
  const double t0 = now_s();
  for (int i = 0; i < n_threads; ++i) {
    worker_arg w = {s, hp, theta, states, actions, returns, B, mode, seconds, 0, P};
    args[i] = w;
    pthread_create(&th[i], NULL, worker, &args[i]);
  }
  long total = 0;
  for (int i = 0; i < n_threads; ++i) {
    pthread_join(th[i], NULL);
    total += args[i].items;
  }
  const double dt = now_s() - t0;
  free(th);
  free(args);
  if (items_done) *items_done = total;
  return (double)total / dt;
}
