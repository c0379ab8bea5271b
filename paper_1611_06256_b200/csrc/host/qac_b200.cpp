// qac_b200.cpp -- reference value-type API (nnet.hpp / returns.hpp) over the
// C ABI.  See qac_b200.hpp for the contract.  Validation runs first, in fp64
// on the host, in the reference's order and with its messages, so the
// exceptions a caller sees are the reference's; the arithmetic then runs on
// the device.
#include "qac_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "ga3c.h"

namespace qac_b200 {
namespace {

thread_local int t_device = 0;

ga3c_net_spec to_c(const nnet::NetworkSpec& s) {
  ga3c_net_spec c{};
  if (s.hidden_dims.size() > GA3C_MAX_HIDDEN || s.conv.size() > GA3C_MAX_CONV)
    throw std::invalid_argument("NetworkSpec: more layers than the device library supports");
  if (s.conv.empty()) {
    c.in_h = 1;
    c.in_w = 1;
    c.in_c = s.input_dim;
  } else {
    const int hw = s.in_h * s.in_w;
    if (s.in_h <= 0 || s.in_w <= 0 || s.input_dim % hw != 0)
      throw std::invalid_argument("NetworkSpec: input_dim is not in_h * in_w * channels");
    c.in_h = s.in_h;
    c.in_w = s.in_w;
    c.in_c = s.input_dim / hw;
  }
  c.n_conv = static_cast<int>(s.conv.size());
  for (int i = 0; i < c.n_conv; ++i) {
    c.conv_out[i] = s.conv[i].out;
    c.conv_k[i] = s.conv[i].k;
    c.conv_stride[i] = s.conv[i].stride;
  }
  c.n_hidden = static_cast<int>(s.hidden_dims.size());
  for (int i = 0; i < c.n_hidden; ++i) c.hidden[i] = s.hidden_dims[i];
  c.n_actions = s.n_actions;
  return c;
}

ga3c_hyper to_c(const nnet::Hyperparams& h) {
  ga3c_hyper c{};
  c.gamma = h.gamma;
  c.t_max = h.t_max;
  c.beta = h.beta;
  c.eps_log = h.eps_log;
  c.eta = h.eta;
  c.alpha = h.alpha;
  c.eps_rms = h.eps_rms;
  c.value_loss_weight = h.value_loss_weight;
  c.grad_clip_norm = h.grad_clip_norm;
  c.clip_rewards = h.clip_rewards ? 1 : 0;
  return c;
}

[[noreturn]] void fail(int st, const char* what) {
  if (st == GA3C_INVALID_ARGUMENT || st == GA3C_NONFINITE_INPUT)
    throw std::invalid_argument(std::string(what) + ": " + ga3c_status_string(st));
  throw std::runtime_error(std::string(what) + ": " + ga3c_status_string(st));
}

void check(int st, const char* what) {
  if (st != GA3C_OK) fail(st, what);
}

// One device model + context per (thread, device, spec, hyperparameters).
// Nothing about theta is cached: every call uploads the caller's values.
struct Entry {
  ga3c_model* m = nullptr;
  ga3c_ctx* c = nullptr;
  int max_batch = 0;
  ~Entry() {
    if (c) ga3c_ctx_destroy(c);
    if (m) ga3c_model_destroy(m);
  }
};

Entry& entry(const ga3c_net_spec& s, const ga3c_hyper& h, int batch) {
  thread_local std::unordered_map<std::string, std::unique_ptr<Entry>> cache;
  std::string key(reinterpret_cast<const char*>(&s), sizeof s);
  key.append(reinterpret_cast<const char*>(&h), sizeof h);
  key.append(reinterpret_cast<const char*>(&t_device), sizeof t_device);
  auto& e = cache[key];
  if (!e) {
    e = std::make_unique<Entry>();
    int st = GA3C_OK;
    e->m = ga3c_model_create(&s, &h, t_device, &st);
    if (!e->m) {
      e.reset();
      fail(st == GA3C_OK ? GA3C_CUDA_ERROR : st, "qac_b200: model create");
    }
  }
  if (batch > e->max_batch) {
    if (e->c) ga3c_ctx_destroy(e->c);
    int mb = 64;
    while (mb < batch) mb *= 2;
    int st = GA3C_OK;
    e->c = ga3c_ctx_create(e->m, mb, &st);
    if (!e->c) {
      e->max_batch = 0;
      fail(st == GA3C_OK ? GA3C_CUDA_ERROR : st, "qac_b200: context create");
    }
    e->max_batch = mb;
  }
  return *e;
}

std::vector<float> to_f32(const std::vector<double>& v) {
  std::vector<float> f(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) f[i] = static_cast<float>(v[i]);
  return f;
}

void check_state(const std::vector<double>& state, int input_dim) {  // nnet.cpp:75-81
  if (static_cast<int>(state.size()) != input_dim)
    throw std::invalid_argument("nnet: state dimension mismatch");
  for (double v : state)
    if (!std::isfinite(v)) throw std::invalid_argument("nnet: non-finite state component");
}

void load(Entry& e, const std::vector<double>& theta, const std::vector<double>* g,
          std::uint64_t version) {
  const std::vector<float> t32 = to_f32(theta);
  std::vector<float> g32;
  if (g) g32 = to_f32(*g);
  check(ga3c_model_load(e.m, t32.data(), g ? g32.data() : nullptr, version), "qac_b200: load");
}

std::vector<float> pack_states(std::span<const std::vector<double>> states, int dim) {
  std::vector<float> x(states.size() * static_cast<std::size_t>(dim));
  for (std::size_t b = 0; b < states.size(); ++b)
    for (int i = 0; i < dim; ++i) x[b * dim + i] = static_cast<float>(states[b][i]);
  return x;
}

}  // namespace

namespace returns {

std::vector<double> compute_returns(std::span<const double> rewards, bool terminal,
                                    double bootstrap_value, double gamma) {
  // returns.cpp:10-17, same order and messages
  if (rewards.empty()) throw std::invalid_argument("compute_returns: empty reward sequence");
  if (!(gamma > 0.0) || gamma > 1.0)
    throw std::invalid_argument("compute_returns: gamma must be in (0, 1]");
  for (double r : rewards)
    if (!std::isfinite(r)) throw std::invalid_argument("compute_returns: non-finite reward");
  if (!terminal && !std::isfinite(bootstrap_value))
    throw std::invalid_argument("compute_returns: non-finite bootstrap value");
  // Any valid spec works: the returns kernel does not touch parameters.
  nnet::NetworkSpec tiny;
  tiny.input_dim = 1;
  tiny.n_actions = 2;
  Entry& e = entry(to_c(tiny), to_c(nnet::Hyperparams{}), 1);
  std::vector<double> out(rewards.size());
  const int32_t off[2] = {0, static_cast<int32_t>(rewards.size())};
  const uint8_t term = terminal ? 1 : 0;
  const double boot = terminal ? 0.0 : bootstrap_value;
  check(ga3c_compute_returns(e.c, rewards.data(), off, 1, &term, &boot, gamma, out.data()),
        "compute_returns");
  return out;
}

}  // namespace returns

namespace nnet {

void set_device(int device) { t_device = device; }

void validate(const NetworkSpec& spec) {  // nnet.cpp:123-130 (+ conv rules)
  if (spec.input_dim <= 0) throw std::invalid_argument("NetworkSpec: input_dim must be positive");
  if (spec.n_actions < 2) throw std::invalid_argument("NetworkSpec: need at least two actions");
  for (int h : spec.hidden_dims)
    if (h <= 0) throw std::invalid_argument("NetworkSpec: hidden dims must be positive");
  const ga3c_net_spec c = to_c(spec);
  if (ga3c_validate_spec(&c) != GA3C_OK)
    throw std::invalid_argument("NetworkSpec: conv stack does not fit the input");
}

void validate(const Hyperparams& hp) {  // nnet.cpp:131-145
  const ga3c_hyper c = to_c(hp);
  if (ga3c_validate_hyper(&c) != GA3C_OK) {
    // re-derive the reference's message
    if (!(hp.gamma > 0.0) || hp.gamma > 1.0)
      throw std::invalid_argument("Hyperparams: gamma must be in (0, 1]");
    if (hp.t_max < 1) throw std::invalid_argument("Hyperparams: t_max must be >= 1");
    if (hp.beta < 0.0) throw std::invalid_argument("Hyperparams: beta must be >= 0");
    if (!(hp.eps_log > 0.0)) throw std::invalid_argument("Hyperparams: eps_log must be > 0");
    if (!(hp.eta > 0.0)) throw std::invalid_argument("Hyperparams: eta must be > 0");
    if (!(hp.alpha >= 0.0) || hp.alpha >= 1.0)
      throw std::invalid_argument("Hyperparams: alpha must be in [0, 1)");
    if (!(hp.eps_rms > 0.0)) throw std::invalid_argument("Hyperparams: eps_rms must be > 0");
    if (hp.value_loss_weight < 0.0)
      throw std::invalid_argument("Hyperparams: value_loss_weight must be >= 0");
    throw std::invalid_argument("Hyperparams: grad_clip_norm must be >= 0");
  }
}

std::size_t param_count(const NetworkSpec& spec) {
  validate(spec);
  const ga3c_net_spec c = to_c(spec);
  return ga3c_param_count(&c);
}

ModelState init_model(const NetworkSpec& spec, std::uint64_t seed) {
  ModelState m;
  m.theta.assign(param_count(spec), 0.0);
  const ga3c_net_spec c = to_c(spec);
  check(ga3c_init_params(&c, seed, m.theta.data(), nullptr), "init_model");
  return m;
}

RmsState init_rms(const NetworkSpec& spec) { return RmsState{std::vector<double>(param_count(spec), 0.0)}; }

double policy_entropy(std::span<const double> policy, double eps_log) {  // nnet.cpp:193-199
  double h = 0.0;
  for (double p : policy)
    if (p > 0.0 || eps_log > 0.0) h -= p * std::log(p + eps_log);
  return h;
}

ForwardResult forward(const ModelState& model, const NetworkSpec& spec,
                      std::span<const std::vector<double>> states) {
  const std::size_t P = param_count(spec);
  if (model.theta.size() != P) throw std::invalid_argument("forward: theta size does not match spec");
  for (const auto& s : states) check_state(s, spec.input_dim);
  ForwardResult out;
  if (states.empty()) return out;
  const int B = static_cast<int>(states.size());
  const ga3c_net_spec cs = to_c(spec);
  Entry& e = entry(cs, to_c(Hyperparams{}), B);
  load(e, model.theta, nullptr, model.version);
  const std::vector<float> x = pack_states(states, spec.input_dim);
  const int A = spec.n_actions;
  // the device's fp64 softmax: rows sum to 1 in fp64 and sample_index on
  // them matches the on-device sampler (util.hpp:46-54)
  std::vector<double> pi(static_cast<std::size_t>(B) * A), v(B);
  check(ga3c_forward64_f32(e.c, -1, x.data(), B, pi.data(), v.data(), nullptr), "forward");
  out.policies.resize(B);
  out.values.resize(B);
  for (int b = 0; b < B; ++b) {
    out.policies[b].assign(pi.begin() + static_cast<std::ptrdiff_t>(b) * A,
                           pi.begin() + static_cast<std::ptrdiff_t>(b + 1) * A);
    out.values[b] = v[b];
  }
  return out;
}

GradientPacket loss_and_gradients(const ModelState& model, const NetworkSpec& spec,
                                  const Hyperparams& hp, const returns::ExperienceBatch& batch) {
  // nnet.cpp:203-228, same order and messages
  validate(spec);
  validate(hp);
  const std::size_t P = param_count(spec);
  if (model.theta.size() != P)
    throw std::invalid_argument("loss_and_gradients: theta size does not match spec");
  if (batch.experiences.empty()) throw std::invalid_argument("loss_and_gradients: empty batch");
  if (batch.returns.size() != batch.experiences.size())
    throw std::invalid_argument("loss_and_gradients: returns/experiences length mismatch");
  const int B = static_cast<int>(batch.experiences.size());
  std::vector<int32_t> actions(B);
  for (int n = 0; n < B; ++n) {
    const auto& e = batch.experiences[n];
    if (!std::isfinite(batch.returns[n]))
      throw std::invalid_argument("loss_and_gradients: non-finite return");
    check_state(e.state, spec.input_dim);
    if (e.action < 0 || e.action >= spec.n_actions)
      throw std::invalid_argument("loss_and_gradients: action out of range");
    actions[n] = e.action;
  }
  const ga3c_net_spec cs = to_c(spec);
  Entry& e = entry(cs, to_c(hp), B);
  load(e, model.theta, nullptr, model.version);
  std::vector<float> x(static_cast<std::size_t>(B) * spec.input_dim);
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < spec.input_dim; ++i)
      x[static_cast<std::size_t>(b) * spec.input_dim + i] = static_cast<float>(batch.experiences[b].state[i]);
  std::vector<float> d(P);
  double sc[3] = {0, 0, 0};
  check(ga3c_loss_grad_f32(e.c, -1, x.data(), actions.data(), batch.returns.data(), B, 1, d.data(), sc),
        "loss_and_gradients");
  GradientPacket pkt;
  pkt.dtheta.assign(d.begin(), d.end());
  pkt.policy_loss = sc[0];
  pkt.value_loss = sc[1];
  pkt.entropy = sc[2];
  pkt.batch_size = B;
  return pkt;
}

UpdateResult rmsprop_update(const ModelState& model, const RmsState& rms, const GradientPacket& grads,
                            const Hyperparams& hp) {
  validate(hp);  // nnet.cpp:295-301
  if (grads.dtheta.size() != model.theta.size() || rms.g.size() != model.theta.size())
    throw std::invalid_argument("rmsprop_update: size mismatch");
  for (double g : grads.dtheta)
    if (!std::isfinite(g)) return UpdateResult{model, rms, false};
  // RMSProp is elementwise over the flat vector: no network layout needed
  const std::size_t P = model.theta.size();
  if (P == 0) return UpdateResult{model, rms, true};
  const ga3c_hyper h = to_c(hp);
  std::vector<float> t32(P), g32(P), d32(P);
  for (std::size_t i = 0; i < P; ++i) {
    t32[i] = static_cast<float>(model.theta[i]);
    g32[i] = static_cast<float>(rms.g[i]);
    d32[i] = static_cast<float>(grads.dtheta[i]);
  }
  int applied = 0;
  const int st = ga3c_rmsprop_flat(&h, t_device, P, t32.data(), g32.data(), d32.data(), &applied);
  if (st == GA3C_NOT_APPLIED || !applied) return UpdateResult{model, rms, false};
  check(st, "rmsprop_update");
  UpdateResult r;
  r.model.theta.assign(t32.begin(), t32.end());
  r.rms.g.assign(g32.begin(), g32.end());
  r.model.version = model.version + 1;
  r.applied = true;
  return r;
}

}  // namespace nnet
}  // namespace qac_b200
