// layout.cpp -- spec validation, parameter layout and seeded init.
#include "layout.hpp"

#include <cmath>
#include <cstring>
#include <random>

namespace ga3c {

// nnet.cpp:123-130, plus VALID conv geometry.
int validate_spec(const ga3c_net_spec& s) {
  if (s.in_h <= 0 || s.in_w <= 0 || s.in_c <= 0) return GA3C_INVALID_ARGUMENT;
  if (s.n_actions < 2) return GA3C_INVALID_ARGUMENT;
  if (s.n_conv < 0 || s.n_conv > GA3C_MAX_CONV) return GA3C_INVALID_ARGUMENT;
  if (s.n_hidden < 0 || s.n_hidden > GA3C_MAX_HIDDEN) return GA3C_INVALID_ARGUMENT;
  int h = s.in_h, w = s.in_w;
  for (int i = 0; i < s.n_conv; ++i) {
    if (s.conv_out[i] <= 0 || s.conv_k[i] <= 0 || s.conv_stride[i] <= 0)
      return GA3C_INVALID_ARGUMENT;
    if (s.conv_k[i] > h || s.conv_k[i] > w) return GA3C_INVALID_ARGUMENT;
    h = (h - s.conv_k[i]) / s.conv_stride[i] + 1;
    w = (w - s.conv_k[i]) / s.conv_stride[i] + 1;
  }
  for (int i = 0; i < s.n_hidden; ++i)
    if (s.hidden[i] <= 0) return GA3C_INVALID_ARGUMENT;
  return GA3C_OK;
}

// nnet.cpp:131-145
int validate_hyper(const ga3c_hyper& hp) {
  if (!(hp.gamma > 0.0) || hp.gamma > 1.0) return GA3C_INVALID_ARGUMENT;
  if (hp.t_max < 1) return GA3C_INVALID_ARGUMENT;
  if (hp.beta < 0.0) return GA3C_INVALID_ARGUMENT;
  if (!(hp.eps_log > 0.0)) return GA3C_INVALID_ARGUMENT;
  if (!(hp.eta > 0.0)) return GA3C_INVALID_ARGUMENT;
  if (!(hp.alpha >= 0.0) || hp.alpha >= 1.0) return GA3C_INVALID_ARGUMENT;
  if (!(hp.eps_rms > 0.0)) return GA3C_INVALID_ARGUMENT;
  if (hp.value_loss_weight < 0.0) return GA3C_INVALID_ARGUMENT;
  if (hp.grad_clip_norm < 0.0) return GA3C_INVALID_ARGUMENT;
  return GA3C_OK;
}

// nnet.cpp:29-45 with conv layers in front.
Layout layout_of(const ga3c_net_spec& s) {
  Layout lo;
  std::size_t off = 0;
  int h = s.in_h, w = s.in_w, c = s.in_c;
  lo.in_dim = h * w * c;
  lo.n_actions = s.n_actions;
  for (int i = 0; i < s.n_conv; ++i) {
    Layer& L = lo.trunk[lo.n_trunk++];
    L.is_conv = true;
    L.cin = c;
    L.cout = s.conv_out[i];
    L.k = s.conv_k[i];
    L.stride = s.conv_stride[i];
    L.ih = h;
    L.iw = w;
    L.oh = (h - L.k) / L.stride + 1;
    L.ow = (w - L.k) / L.stride + 1;
    L.in = L.k * L.k * c;
    L.out = L.cout;
    L.w_off = off;
    L.b_off = off + static_cast<std::size_t>(L.cout) * L.in;
    off = L.b_off + L.cout;
    h = L.oh;
    w = L.ow;
    c = L.cout;
  }
  lo.n_conv = lo.n_trunk;
  int prev = h * w * c;
  for (int i = 0; i < s.n_hidden; ++i) {
    Layer& L = lo.trunk[lo.n_trunk++];
    L.in = prev;
    L.out = s.hidden[i];
    L.w_off = off;
    L.b_off = off + static_cast<std::size_t>(prev) * L.out;
    off = L.b_off + L.out;
    prev = L.out;
  }
  lo.policy.in = prev;
  lo.policy.out = s.n_actions;
  lo.policy.w_off = off;
  lo.policy.b_off = off + static_cast<std::size_t>(prev) * s.n_actions;
  off = lo.policy.b_off + s.n_actions;
  lo.value.in = prev;
  lo.value.out = 1;
  lo.value.w_off = off;
  lo.value.b_off = off + prev;
  off = lo.value.b_off + 1;
  lo.total = off;
  return lo;
}

std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// nnet.cpp:152-168: U(+-1/sqrt(fan_in)) in layout order, biases zero.
void init_params(const Layout& lo, std::uint64_t seed, double* theta) {
  std::memset(theta, 0, lo.total * sizeof(double));
  std::mt19937_64 rng(seed);
  auto fill = [&](const Layer& L) {
    const double bound = 1.0 / std::sqrt(static_cast<double>(L.in));
    const std::size_t n = static_cast<std::size_t>(L.in) * L.out;
    for (std::size_t i = 0; i < n; ++i)
      theta[L.w_off + i] = (static_cast<double>(rng() >> 11) * 0x1.0p-53 * 2.0 - 1.0) * bound;
  };
  for (int i = 0; i < lo.n_trunk; ++i) fill(lo.trunk[i]);
  fill(lo.policy);
  fill(lo.value);
}

}  // namespace ga3c
