// test_qac_adapter.cpp -- the reference's own nnet / returns unit tests
// (proj/tests/test_nnet.cpp, test_returns.cpp) restated against the B200
// drop-in adapter (include/qac_b200.hpp), compiled the way a reference
// caller is: `#include "qac/nnet.hpp"` resolves to the shim in include/qac/,
// so `qac::nnet::forward` etc. are the device implementation.  Exact fp64 expectations of the reference become
// fp32 tolerances; returns stay bitwise.  Needs a GPU; built
// and run by tests/test_qac_adapter_gpu.py.
#include "qac/nnet.hpp"
#include "qac/returns.hpp"

#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

using qac::nnet::ForwardResult;
using qac::nnet::GradientPacket;
using qac::nnet::Hyperparams;
using qac::nnet::ModelState;
using qac::nnet::NetworkSpec;
using qac::returns::Experience;
using qac::returns::ExperienceBatch;
namespace nnet = qac::nnet;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                               \
  do {                                                         \
    ++g_checks;                                                \
    if (!(c)) {                                                \
      ++g_fail;                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                          \
  } while (0)
#define CHECK_THROWS_INVALID(expr)              \
  do {                                          \
    bool threw_ = false;                        \
    try {                                       \
      (void)(expr);                             \
    } catch (const std::invalid_argument&) {    \
      threw_ = true;                            \
    }                                           \
    CHECK(threw_);                              \
  } while (0)

static double next_uniform(std::mt19937_64& rng) {  // util.hpp:41-43
  return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}

static NetworkSpec mlp(int in, std::vector<int> hidden, int a) {
  NetworkSpec s;
  s.input_dim = in;
  s.hidden_dims = std::move(hidden);
  s.n_actions = a;
  return s;
}

static ExperienceBatch random_batch(const NetworkSpec& spec, int n, std::uint64_t seed) {  // test_nnet.cpp:43-55
  std::mt19937_64 rng(seed);
  ExperienceBatch batch;
  for (int i = 0; i < n; ++i) {
    Experience e;
    e.state.resize(static_cast<std::size_t>(spec.input_dim));
    for (double& x : e.state) x = next_uniform(rng) * 2.0 - 1.0;
    e.action = static_cast<int>(next_uniform(rng) * spec.n_actions);
    batch.experiences.push_back(std::move(e));
    batch.returns.push_back(next_uniform(rng) * 4.0 - 2.0);
  }
  return batch;
}

static void param_counts() {  // test_nnet.cpp:99-106
  CHECK(nnet::param_count(mlp(4, {8}, 3)) == 76);
  CHECK(nnet::param_count(mlp(2, {}, 2)) == 2 * 2 + 2 + 2 + 1);
  CHECK(nnet::param_count(mlp(5, {7, 3}, 4)) == (5 * 7 + 7) + (7 * 3 + 3) + (3 * 4 + 4) + (3 + 1));
  NetworkSpec a = mlp(84 * 84 * 4, {256}, 6);  // DNN A
  a.in_h = a.in_w = 84;
  a.conv = {{16, 8, 4}, {32, 4, 2}};
  CHECK(nnet::param_count(a) == 677943);
}

static void init_deterministic() {  // test_nnet.cpp:108-125
  const NetworkSpec spec = mlp(4, {8}, 3);
  const auto a = nnet::init_model(spec, 7), b = nnet::init_model(spec, 7), c = nnet::init_model(spec, 8);
  CHECK(a.theta == b.theta);
  CHECK(a.theta != c.theta);
  CHECK(a.version == 0);
  for (int i = 0; i < 32; ++i) CHECK(std::abs(a.theta[i]) <= 0.5);
  for (int i = 32; i < 40; ++i) CHECK(a.theta[i] == 0.0);
  const double hb = 1.0 / std::sqrt(8.0);
  for (int i = 40; i < 64; ++i) CHECK(std::abs(a.theta[i]) <= hb);
  for (int i = 64; i < 67; ++i) CHECK(a.theta[i] == 0.0);
  for (int i = 67; i < 75; ++i) CHECK(std::abs(a.theta[i]) <= hb);
  CHECK(a.theta[75] == 0.0);
}

static void forward_simplex_and_validation() {  // test_nnet.cpp:127-152
  const NetworkSpec spec = mlp(4, {8}, 3);
  auto model = nnet::init_model(spec, 3);
  for (double& t : model.theta) t *= 50.0;  // extreme logits saturate, never overflow
  std::vector<std::vector<double>> states{{1, 2, 3, 4}, {-1e3, 5e2, 0, 1}, {0, 0, 0, 0}};
  const auto fr = nnet::forward(model, spec, states);
  CHECK(fr.policies.size() == 3);
  for (const auto& pi : fr.policies) {
    double sum = 0.0;
    for (double p : pi) {
      CHECK(std::isfinite(p));
      CHECK(p >= 0.0);
      sum += p;
    }
    CHECK(std::abs(sum - 1.0) < 1e-6);
  }
  for (double v : fr.values) CHECK(std::isfinite(v));
  std::vector<std::vector<double>> wrong{{1, 2, 3}};
  CHECK_THROWS_INVALID(nnet::forward(model, spec, wrong));
  std::vector<std::vector<double>> nan{{1, std::nan(""), 3, 4}};
  CHECK_THROWS_INVALID(nnet::forward(model, spec, nan));
  ModelState bad = model;
  bad.theta.pop_back();
  CHECK_THROWS_INVALID(nnet::forward(bad, spec, states));
  CHECK(nnet::forward(model, spec, std::vector<std::vector<double>>{}).values.empty());
}

// test_nnet.cpp:154-173: the reference checks against central differences at
// h = 1e-5 in fp64.  The device is fp32, so the loss is evaluated on the
// host in fp64 from device forwards (frozen advantage) at a larger step.
static void gradients_match_finite_differences() {
  const NetworkSpec spec = mlp(6, {8}, 3);
  Hyperparams hp;
  const auto batch = random_batch(spec, 4, 99);
  const ModelState model = nnet::init_model(spec, 5);
  std::vector<std::vector<double>> states;
  for (const auto& e : batch.experiences) states.push_back(e.state);
  const auto base = nnet::forward(model, spec, states);
  std::vector<double> adv(states.size());
  for (std::size_t i = 0; i < adv.size(); ++i) adv[i] = batch.returns[i] - base.values[i];
  auto loss = [&](const ModelState& m) {
    const auto fr = nnet::forward(m, spec, states);
    double L = 0.0;
    for (std::size_t n = 0; n < states.size(); ++n) {
      const auto& pi = fr.policies[n];
      double H = 0.0;
      for (double p : pi) H -= p * std::log(p + hp.eps_log);
      L += -std::log(pi[batch.experiences[n].action] + hp.eps_log) * adv[n] - hp.beta * H;
      const double d = batch.returns[n] - fr.values[n];
      L += hp.value_loss_weight * d * d;
    }
    return L;
  };
  const auto pkt = nnet::loss_and_gradients(model, spec, hp, batch);
  CHECK(pkt.dtheta.size() == model.theta.size());
  double gmax = 0.0;
  for (double g : pkt.dtheta) gmax = std::max(gmax, std::abs(g));
  double worst = 0.0;
  for (std::size_t i = 0; i < model.theta.size(); ++i) {
    const double h = 2e-3;
    ModelState p = model, m = model;
    p.theta[i] += h;
    m.theta[i] -= h;
    const double fd = (loss(p) - loss(m)) / (2 * h);
    worst = std::max(worst, std::abs(fd - pkt.dtheta[i]) / gmax);
  }
  if (worst >= 2e-3) std::printf("fd worst %g\n", worst);
  CHECK(worst < 2e-3);
}

static void gradients_summed() {  // test_nnet.cpp:175-189
  const NetworkSpec spec = mlp(4, {8}, 3);
  const Hyperparams hp;
  const auto model = nnet::init_model(spec, 11);
  auto one = random_batch(spec, 1, 12);
  auto two = one;
  two.experiences.push_back(one.experiences[0]);
  two.returns.push_back(one.returns[0]);
  const auto a = nnet::loss_and_gradients(model, spec, hp, one);
  const auto b = nnet::loss_and_gradients(model, spec, hp, two);
  for (std::size_t i = 0; i < a.dtheta.size(); ++i)
    CHECK(std::abs(b.dtheta[i] - 2.0 * a.dtheta[i]) <= 1e-6 * std::abs(a.dtheta[i]) + 1e-12);
  CHECK(b.batch_size == 2);
}

static void collapsed_policy_finite() {  // test_nnet.cpp:191-227
  const NetworkSpec spec = mlp(2, {}, 2);
  const Hyperparams hp;
  ModelState model = nnet::init_model(spec, 1);
  // policy W rows: push action 0 to probability ~0
  model.theta[0] = -40.0;
  model.theta[1] = -40.0;
  model.theta[2] = 40.0;
  model.theta[3] = 40.0;
  ExperienceBatch b;
  Experience e;
  e.state = {1.0, 1.0};
  e.action = 0;
  b.experiences.push_back(e);
  b.returns.push_back(1.0);
  const auto fr = nnet::forward(model, spec, std::vector<std::vector<double>>{e.state});
  CHECK(fr.policies[0][0] < 1e-15);
  const auto pkt = nnet::loss_and_gradients(model, spec, hp, b);
  for (double g : pkt.dtheta) CHECK(std::isfinite(g));
}

static void entropy_helper() {  // test_nnet.cpp:229-235
  const std::vector<double> uniform{0.25, 0.25, 0.25, 0.25}, collapsed{1, 0, 0, 0};
  CHECK(std::abs(nnet::policy_entropy(uniform, 0.0) - std::log(4.0)) < 1e-12);
  CHECK(nnet::policy_entropy(collapsed, 0.0) == 0.0);
  CHECK(std::isfinite(nnet::policy_entropy(collapsed, 1e-6)));
}

static void rmsprop_arithmetic() {  // test_nnet.cpp:237-274, fp32 device arithmetic
  const NetworkSpec spec = mlp(1, {}, 2);
  Hyperparams hp;
  hp.alpha = 0.99;
  hp.eta = 0.1;
  hp.eps_rms = 1e-8;
  ModelState model;
  model.theta.assign(nnet::param_count(spec), 0.0);
  model.theta[0] = 1.0;
  auto rms = nnet::init_rms(spec);
  GradientPacket pkt;
  pkt.dtheta.assign(model.theta.size(), 0.0);
  pkt.dtheta[0] = 2.0;
  const auto res = nnet::rmsprop_update(model, rms, pkt, hp);
  CHECK(res.applied);
  const double g = 0.99 * 0.0 + (1.0 - 0.99) * 2.0 * 2.0;
  const double expect = 1.0 - 0.1 * 2.0 / std::sqrt(g + 1e-8);
  CHECK(std::abs(res.rms.g[0] - g) <= 1e-6 * g);
  CHECK(std::abs(res.model.theta[0] - expect) <= 1e-6);
  CHECK(res.model.version == 1);
  CHECK(res.model.theta[1] == 0.0);
  GradientPacket pkt2;
  pkt2.dtheta.assign(model.theta.size(), 0.0);
  pkt2.dtheta[0] = -1.0;
  const auto res2 = nnet::rmsprop_update(res.model, res.rms, pkt2, hp);
  const double g2 = 0.99 * g + (1.0 - 0.99);
  const double expect2 = expect + 0.1 / std::sqrt(g2 + 1e-8);
  CHECK(std::abs(res2.rms.g[0] - g2) <= 1e-6 * g2);
  CHECK(std::abs(res2.model.theta[0] - expect2) <= 1e-6);
  CHECK(res2.model.version == 2);
}

static void rmsprop_rejects_nonfinite() {  // test_nnet.cpp:276-291 (bitwise: inputs unchanged)
  const NetworkSpec spec = mlp(2, {}, 2);
  const Hyperparams hp;
  const auto model = nnet::init_model(spec, 3);
  auto rms = nnet::init_rms(spec);
  rms.g[0] = 0.5;
  GradientPacket pkt;
  pkt.dtheta.assign(model.theta.size(), 0.0);
  pkt.dtheta[1] = std::numeric_limits<double>::quiet_NaN();
  const auto res = nnet::rmsprop_update(model, rms, pkt, hp);
  CHECK(!res.applied);
  CHECK(res.model.theta == model.theta);
  CHECK(res.model.version == model.version);
  CHECK(res.rms.g == rms.g);
}

static void gradient_clip() {  // test_nnet.cpp:293-313
  const NetworkSpec spec = mlp(4, {8}, 3);
  Hyperparams hp;
  const auto model = nnet::init_model(spec, 21);
  const auto batch = random_batch(spec, 5, 22);
  const auto raw = nnet::loss_and_gradients(model, spec, hp, batch);
  double norm = 0.0;
  for (double g : raw.dtheta) norm += g * g;
  CHECK(std::sqrt(norm) > 0.02);
  hp.grad_clip_norm = 0.01;
  const auto clipped = nnet::loss_and_gradients(model, spec, hp, batch);
  double cn = 0.0;
  for (double g : clipped.dtheta) cn += g * g;
  CHECK(std::abs(std::sqrt(cn) - 0.01) <= 1e-7);
  CHECK(clipped.dtheta[0] * raw.dtheta[0] >= 0.0);
}

static void loss_validation() {  // test_nnet.cpp:315-330
  const NetworkSpec spec = mlp(2, {}, 2);
  const Hyperparams hp;
  const auto model = nnet::init_model(spec, 1);
  ExperienceBatch empty;
  CHECK_THROWS_INVALID(nnet::loss_and_gradients(model, spec, hp, empty));
  auto b = random_batch(spec, 2, 3);
  auto mism = b;
  mism.returns.pop_back();
  CHECK_THROWS_INVALID(nnet::loss_and_gradients(model, spec, hp, mism));
  auto bad_a = b;
  bad_a.experiences[1].action = 2;
  CHECK_THROWS_INVALID(nnet::loss_and_gradients(model, spec, hp, bad_a));
  auto bad_r = b;
  bad_r.returns[0] = std::numeric_limits<double>::infinity();
  CHECK_THROWS_INVALID(nnet::loss_and_gradients(model, spec, hp, bad_r));
  Hyperparams bad_hp;
  bad_hp.gamma = 0.0;
  CHECK_THROWS_INVALID(nnet::loss_and_gradients(model, spec, bad_hp, b));
  CHECK_THROWS_INVALID(nnet::param_count(mlp(2, {}, 1)));
}

static std::vector<double> host_returns(const std::vector<double>& r, bool term, double boot, double gamma) {
  std::vector<double> out(r.size());
  double acc = term ? 0.0 : boot;
  for (std::size_t i = r.size(); i-- > 0;) {
    acc = r[i] + gamma * acc;
    out[i] = acc;
  }
  return out;
}

static void returns_known_answers() {  // test_returns.cpp:37-84, bitwise
  using qac::returns::compute_returns;
  const auto r = compute_returns(std::vector<double>{1, 0, 0, 1}, true, 123.0, 0.99);
  CHECK(r == host_returns({1, 0, 0, 1}, true, 0, 0.99));
  CHECK(std::abs(r[0] - (1.0 + 0.99 * 0.9801)) <= 1e-15);
  const auto b = compute_returns(std::vector<double>{0, 0}, false, 10.0, 0.5);
  CHECK(b[0] == 2.5 && b[1] == 5.0);
  CHECK(compute_returns(std::vector<double>{0.3, -1.2, 8.0}, true, 0.0, 0.9) ==
        compute_returns(std::vector<double>{0.3, -1.2, 8.0}, true, 1e9, 0.9));
  const auto g1 = compute_returns(std::vector<double>{1, 1, 1}, true, 0.0, 1.0);
  CHECK(g1[0] == 3.0 && g1[1] == 2.0 && g1[2] == 1.0);
  std::mt19937_64 rng(42);
  for (int t = 0; t < 200; ++t) {
    const std::size_t n = 1 + static_cast<std::size_t>(next_uniform(rng) * 20.0);
    std::vector<double> rw(n);
    for (double& x : rw) x = next_uniform(rng) * 20.0 - 10.0;
    const bool term = next_uniform(rng) < 0.5;
    const double boot = next_uniform(rng) * 10.0 - 5.0;
    const double gamma = 0.5 + next_uniform(rng) * 0.5;
    CHECK(compute_returns(rw, term, boot, gamma) == host_returns(rw, term, boot, gamma));
  }
  CHECK_THROWS_INVALID(compute_returns(std::vector<double>{}, true, 0.0, 0.9));
  CHECK_THROWS_INVALID(compute_returns(std::vector<double>{1.0}, true, 0.0, 0.0));
  CHECK_THROWS_INVALID(compute_returns(std::vector<double>{std::nan("")}, true, 0.0, 0.9));
  CHECK_THROWS_INVALID(compute_returns(std::vector<double>{1.0}, false, std::nan(""), 0.9));
}

static void dnn_a_concurrent_callers() {
  // pipeline.cpp:65-93: several predictor threads call forward concurrently on
  // one model; every thread must see the same answer.
  NetworkSpec spec = mlp(84 * 84 * 4, {256}, 6);
  spec.in_h = spec.in_w = 84;
  spec.conv = {{16, 8, 4}, {32, 4, 2}};
  const auto model = nnet::init_model(spec, 1);
  std::mt19937_64 rng(5);
  std::vector<std::vector<double>> states(8, std::vector<double>(spec.input_dim));
  for (auto& s : states)
    for (double& x : s) x = static_cast<double>(rng() >> 56) / 256.0;
  const auto ref = nnet::forward(model, spec, states);
  std::vector<ForwardResult> got(4);
  std::vector<std::thread> th;
  for (int t = 0; t < 4; ++t) th.emplace_back([&, t] { got[t] = nnet::forward(model, spec, states); });
  for (auto& t : th) t.join();
  for (const auto& g : got) {
    CHECK(g.values == ref.values);
    CHECK(g.policies == ref.policies);
  }
  ExperienceBatch b;
  for (int i = 0; i < 8; ++i) {
    Experience e;
    e.state = states[i];
    e.action = i % 6;
    b.experiences.push_back(e);
    b.returns.push_back(0.25 * i - 1.0);
  }
  const auto pkt = nnet::loss_and_gradients(model, spec, Hyperparams{}, b);
  double n2 = 0.0;
  for (double g : pkt.dtheta) n2 += g * g;
  CHECK(std::isfinite(n2) && n2 > 0.0);
  CHECK(pkt.batch_size == 8);
}

int main() {
  param_counts();
  init_deterministic();
  forward_simplex_and_validation();
  gradients_match_finite_differences();
  gradients_summed();
  collapsed_policy_finite();
  entropy_helper();
  rmsprop_arithmetic();
  rmsprop_rejects_nonfinite();
  gradient_clip();
  loss_validation();
  returns_known_answers();
  dnn_a_concurrent_callers();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
