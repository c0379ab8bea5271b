// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" face over the UNMODIFIED reference sources
// /root/reference/proj/src/{nnet,returns}.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/libqac_ref.so.  Nothing here restates the
// algorithm: each entry point marshals flat arrays into the reference's own
// value types and calls the reference function named in its comment.  It is
// used to pin oracle/ga3c_oracle.c bit for bit on MLP specs and to produce the
// golden vectors under tests/golden/ (tests/golden/make_golden.py).
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "ga3c_oracle.h"
#include "qac/nnet.hpp"
#include "qac/returns.hpp"
#include "qac/util.hpp"

using namespace qac;

namespace {

nnet::NetworkSpec to_spec(int input_dim, const int* hidden, int n_hidden, int n_actions) {
  nnet::NetworkSpec s;
  s.input_dim = input_dim;
  s.hidden_dims.assign(hidden, hidden + n_hidden);
  s.n_actions = n_actions;
  return s;
}

nnet::Hyperparams to_hyper(const orc_hyper* h) {
  nnet::Hyperparams hp;
  hp.gamma = h->gamma;
  hp.t_max = h->t_max;
  hp.beta = h->beta;
  hp.eps_log = h->eps_log;
  hp.eta = h->eta;
  hp.alpha = h->alpha;
  hp.eps_rms = h->eps_rms;
  hp.value_loss_weight = h->value_loss_weight;
  hp.grad_clip_norm = h->grad_clip_norm;
  hp.clip_rewards = h->clip_rewards != 0;
  return hp;
}

}  // namespace

extern "C" {

// nnet::param_count (nnet.hpp:71); 0 on std::invalid_argument
size_t ref_param_count(int input_dim, const int* hidden, int n_hidden, int n_actions) {
  try {
    return nnet::param_count(to_spec(input_dim, hidden, n_hidden, n_actions));
  } catch (const std::invalid_argument&) {
    return 0;
  }
}

// nnet::init_model (nnet.hpp:75)
int ref_init_model(int input_dim, const int* hidden, int n_hidden, int n_actions, uint64_t seed,
                   double* theta) {
  try {
    auto m = nnet::init_model(to_spec(input_dim, hidden, n_hidden, n_actions), seed);
    std::memcpy(theta, m.theta.data(), m.theta.size() * sizeof(double));
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

// nnet::forward (nnet.hpp:81)
int ref_forward(int input_dim, const int* hidden, int n_hidden, int n_actions, const double* theta,
                size_t P, const double* states, int B, double* pi, double* v) {
  try {
    auto spec = to_spec(input_dim, hidden, n_hidden, n_actions);
    nnet::ModelState m;
    m.theta.assign(theta, theta + P);
    std::vector<std::vector<double>> st;
    for (int b = 0; b < B; ++b)
      st.emplace_back(states + static_cast<size_t>(b) * input_dim,
                      states + static_cast<size_t>(b + 1) * input_dim);
    auto fr = nnet::forward(m, spec, st);
    for (int b = 0; b < B; ++b) {
      std::memcpy(pi + static_cast<size_t>(b) * n_actions, fr.policies[b].data(),
                  sizeof(double) * n_actions);
      v[b] = fr.values[b];
    }
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

// nnet::loss_and_gradients (nnet.hpp:94)
int ref_loss_and_gradients(int input_dim, const int* hidden, int n_hidden, int n_actions,
                           const orc_hyper* h, const double* theta, size_t P, const double* states,
                           const int* actions, const double* rets, int B, double* dtheta,
                           double* scalars) {
  try {
    auto spec = to_spec(input_dim, hidden, n_hidden, n_actions);
    nnet::ModelState m;
    m.theta.assign(theta, theta + P);
    returns::ExperienceBatch batch;
    for (int b = 0; b < B; ++b) {
      returns::Experience e;
      e.state.assign(states + static_cast<size_t>(b) * input_dim,
                     states + static_cast<size_t>(b + 1) * input_dim);
      e.action = actions[b];
      batch.experiences.push_back(std::move(e));
      batch.returns.push_back(rets[b]);
    }
    auto pkt = nnet::loss_and_gradients(m, spec, to_hyper(h), batch);
    std::memcpy(dtheta, pkt.dtheta.data(), sizeof(double) * pkt.dtheta.size());
    scalars[0] = pkt.policy_loss;
    scalars[1] = pkt.value_loss;
    scalars[2] = pkt.entropy;
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

// nnet::rmsprop_update (nnet.hpp:103); returns 1 applied, 0 rejected, -1 invalid
int ref_rmsprop_update(const orc_hyper* h, const double* theta, const double* g,
                       const double* dtheta, size_t P, double* theta_out, double* g_out,
                       uint64_t version_in, uint64_t* version_out) {
  try {
    nnet::ModelState m;
    m.theta.assign(theta, theta + P);
    m.version = version_in;
    nnet::RmsState r;
    r.g.assign(g, g + P);
    nnet::GradientPacket pkt;
    pkt.dtheta.assign(dtheta, dtheta + P);
    auto res = nnet::rmsprop_update(m, r, pkt, to_hyper(h));
    std::memcpy(theta_out, res.model.theta.data(), sizeof(double) * P);
    std::memcpy(g_out, res.rms.g.data(), sizeof(double) * P);
    *version_out = res.model.version;
    return res.applied ? 1 : 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// returns::compute_returns (returns.hpp:31)
int ref_compute_returns(const double* rewards, int n, int terminal, double bootstrap, double gamma,
                        double* out) {
  try {
    auto r = returns::compute_returns(std::span<const double>(rewards, static_cast<size_t>(n)),
                                      terminal != 0, bootstrap, gamma);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

// nnet::policy_entropy (nnet.hpp:86)
double ref_policy_entropy(const double* p, int n, double eps) {
  return nnet::policy_entropy(std::span<const double>(p, static_cast<size_t>(n)), eps);
}

// qac::next_uniform over std::mt19937_64(seed) (util.hpp:41-43)
void ref_uniforms(uint64_t seed, double* out, size_t n) {
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = next_uniform(rng);
}

// qac::sample_index (util.hpp:46-54): n_draws samples from one policy row,
// one rng draw each, from std::mt19937_64(seed)
void ref_sample_many(const double* probs, int n, uint64_t seed, int n_draws, int* out) {
  std::mt19937_64 rng(seed);
  for (int i = 0; i < n_draws; ++i)
    out[i] = sample_index(std::span<const double>(probs, static_cast<size_t>(n)), rng);
}

// qac::derive_seed (util.hpp:28-32)
uint64_t ref_derive_seed(uint64_t base, const uint64_t* salts, int n) {
  uint64_t h = mix64(base);
  for (int i = 0; i < n; ++i) h = mix64(h ^ salts[i]);
  return h;
}

}  // extern "C"
