// envs.cpp -- seeds/sampling (util.hpp), CPU environments (envs.cpp) and the
// knob annealer (annealer.cpp) of the host engine.
//
// The vector environments keep the reference dynamics (envs.cpp:23-164).
// Two pixel environments feed the conv nets with 84x84x4 u8 frames:
//   FrameCatch -- Catch on a G x G grid rendered into 84x84 frames (12 px
//                 cells for G = 7), stacked over the last 4 steps; a small
//                 learnable Atari-style task for DNN A.
//   Frames     -- DelayLab-style throughput ballast with synthetic frames
//                 (busy-wait step, fixed episode length).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "ga3c_host.hpp"

namespace ga3c::host {

// ---------------------------------------------------------------- util
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

std::uint64_t derive_seed(std::uint64_t base, std::initializer_list<std::uint64_t> salts) {
  std::uint64_t h = mix64(base);
  for (std::uint64_t s : salts) h = mix64(h ^ s);
  return h;
}

double next_uniform(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

int sample_index(const double* probs, int n, std::mt19937_64& rng) {
  const double u = next_uniform(rng);
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += probs[i];
    if (u < acc) return i;
  }
  return n - 1;
}

int argmax_index(const double* v, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

void busy_wait_us(std::int64_t us) {
  if (us <= 0) return;
  const auto until = std::chrono::steady_clock::now() + std::chrono::microseconds(us);
  while (std::chrono::steady_clock::now() < until) {
  }
}

// ---------------------------------------------------------------- envs
namespace {

int uniform_int(std::mt19937_64& rng, int n) { return static_cast<int>(next_uniform(rng) * n); }

void check_action(int a, int n) {
  if (a < 0 || a >= n) throw std::invalid_argument("env: action out of range");
}

ga3c_net_spec vec_input(int dim) {
  ga3c_net_spec s{};
  s.in_h = 1;
  s.in_w = 1;
  s.in_c = dim;
  return s;
}

ga3c_net_spec frame_input() {
  ga3c_net_spec s{};
  s.in_h = 84;
  s.in_w = 84;
  s.in_c = 4;
  return s;
}

class BanditEnv final : public Env {  // envs.cpp:23-56
 public:
  explicit BanditEnv(const EnvSpec& s) : s_(s) {}
  Observation reset(std::uint64_t seed) override {
    rng_.seed(mix64(seed));
    ctx_ = uniform_int(rng_, s_.n_contexts);
    done_ = false;
    Observation o;
    o.f32.assign(s_.n_contexts, 0.f);
    o.f32[ctx_] = 1.f;
    return o;
  }
  StepResult step(int a) override {
    if (done_) throw std::logic_error("env: step after terminal");
    check_action(a, s_.n_actions);
    done_ = true;
    StepResult r;
    r.observation.f32.assign(s_.n_contexts, 0.f);
    r.reward = a == ctx_ % s_.n_actions ? 1.0 : 0.0;
    r.terminal = true;
    return r;
  }
  int action_count() const override { return s_.n_actions; }
  bool frames() const override { return false; }
  ga3c_net_spec input() const override { return vec_input(s_.n_contexts); }

 private:
  EnvSpec s_;
  std::mt19937_64 rng_;
  int ctx_ = 0;
  bool done_ = true;
};

class CatchEnv final : public Env {  // envs.cpp:61-103
 public:
  explicit CatchEnv(const EnvSpec& s) : g_(s.grid_size) {}
  Observation reset(std::uint64_t seed) override {
    std::mt19937_64 rng(mix64(seed));
    row_ = 0;
    col_ = uniform_int(rng, g_);
    pad_ = uniform_int(rng, g_);
    done_ = false;
    return observe();
  }
  StepResult step(int a) override {
    if (done_) throw std::logic_error("env: step after terminal");
    check_action(a, 3);
    pad_ = std::clamp(pad_ + (a - 1), 0, g_ - 1);
    row_ += 1;
    StepResult r;
    r.terminal = row_ == g_ - 1;
    r.reward = r.terminal ? (pad_ == col_ ? 1.0 : -1.0) : 0.0;
    done_ = r.terminal;
    r.observation = observe();
    return r;
  }
  int action_count() const override { return 3; }
  bool frames() const override { return false; }
  ga3c_net_spec input() const override { return vec_input(g_ * g_ + g_); }

 private:
  Observation observe() const {
    Observation o;
    o.f32.assign(g_ * g_ + g_, 0.f);
    o.f32[row_ * g_ + col_] = 1.f;
    o.f32[g_ * g_ + pad_] = 1.f;
    return o;
  }
  int g_, row_ = 0, col_ = 0, pad_ = 0;
  bool done_ = true;
};

class DelayLabEnv final : public Env {  // envs.cpp:107-137
 public:
  explicit DelayLabEnv(const EnvSpec& s) : s_(s) {}
  Observation reset(std::uint64_t) override {
    steps_ = 0;
    done_ = false;
    Observation o;
    o.f32.assign(4, 0.f);
    return o;
  }
  StepResult step(int a) override {
    if (done_) throw std::logic_error("env: step after terminal");
    check_action(a, 2);
    busy_wait_us(s_.step_delay_us);
    StepResult r;
    r.observation.f32.assign(4, 0.f);
    r.terminal = ++steps_ >= s_.episode_len;
    done_ = r.terminal;
    return r;
  }
  int action_count() const override { return 2; }
  bool frames() const override { return false; }
  ga3c_net_spec input() const override { return vec_input(4); }

 private:
  EnvSpec s_;
  int steps_ = 0;
  bool done_ = true;
};

constexpr int kFrameBytes = 84 * 84 * 4;

class FrameCatchEnv final : public Env {
 public:
  explicit FrameCatchEnv(const EnvSpec& s) : s_(s), g_(s.grid_size), cell_(84 / s.grid_size) {}
  Observation reset(std::uint64_t seed) override {
    std::mt19937_64 rng(mix64(seed));
    row_ = 0;
    col_ = uniform_int(rng, g_);
    pad_ = uniform_int(rng, g_);
    done_ = false;
    std::memset(stack_, 0, sizeof(stack_));
    for (int k = 0; k < 4; ++k) push_frame();
    return observe();
  }
  StepResult step(int a) override {
    if (done_) throw std::logic_error("env: step after terminal");
    check_action(a, s_.n_actions);
    busy_wait_us(s_.step_delay_us);
    pad_ = std::clamp(pad_ + (a % 3 - 1), 0, g_ - 1);
    row_ += 1;
    StepResult r;
    r.terminal = row_ == g_ - 1;
    r.reward = r.terminal ? (pad_ == col_ ? 1.0 : -1.0) : 0.0;
    done_ = r.terminal;
    push_frame();
    r.observation = observe();
    return r;
  }
  int action_count() const override { return s_.n_actions; }
  bool frames() const override { return true; }
  ga3c_net_spec input() const override { return frame_input(); }
  void set_single_frame(bool on) override { single_ = on; }

 private:
  void push_frame() {  // channel t = frame t of the 4-step stack (NHWC)
    for (int p = 0; p < 84 * 84; ++p)
      for (int c = 0; c < 3; ++c) stack_[p * 4 + c] = stack_[p * 4 + c + 1];
    for (int p = 0; p < 84 * 84; ++p) stack_[p * 4 + 3] = 0;
    auto paint = [&](int gr, int gc, uint8_t v) {
      for (int y = gr * cell_; y < (gr + 1) * cell_; ++y)
        for (int x = gc * cell_; x < (gc + 1) * cell_; ++x) stack_[(y * 84 + x) * 4 + 3] = v;
    };
    paint(row_, col_, 255);
    paint(g_ - 1, pad_, 128);
  }
  Observation observe() const {
    Observation o;
    if (single_) {  // the newest channel
      o.u8.resize(kFrameBytes / 4);
      for (int p = 0; p < 84 * 84; ++p) o.u8[p] = stack_[p * 4 + 3];
    } else {
      o.u8.assign(stack_, stack_ + kFrameBytes);
    }
    return o;
  }
  EnvSpec s_;
  int g_, cell_, row_ = 0, col_ = 0, pad_ = 0;
  bool done_ = true;
  bool single_ = false;
  uint8_t stack_[kFrameBytes];
};

class FramesEnv final : public Env {
 public:
  explicit FramesEnv(const EnvSpec& s) : s_(s) {}
  Observation reset(std::uint64_t seed) override {
    state_ = mix64(seed) | 1ULL;
    steps_ = 0;
    done_ = false;
    return frame();
  }
  StepResult step(int a) override {
    if (done_) throw std::logic_error("env: step after terminal");
    check_action(a, s_.n_actions);
    busy_wait_us(s_.step_delay_us);
    StepResult r;
    r.reward = (a == static_cast<int>(state_ % s_.n_actions)) ? 1.0 : 0.0;
    r.terminal = ++steps_ >= s_.episode_len;
    done_ = r.terminal;
    r.observation = frame();
    return r;
  }
  int action_count() const override { return s_.n_actions; }
  bool frames() const override { return true; }
  ga3c_net_spec input() const override { return frame_input(); }
  void set_single_frame(bool on) override { single_ = on; }

 private:
  // a fresh synthetic state per step (frames mode), or a fresh newest frame
  // (single-frame mode, stacked on the device)
  Observation frame() {
    Observation o;
    const int bytes = single_ ? kFrameBytes / 4 : kFrameBytes;
    o.u8.resize(bytes);
    std::uint64_t* w = reinterpret_cast<std::uint64_t*>(o.u8.data());
    for (int i = 0; i < bytes / 8; ++i) {  // xorshift64*
      state_ ^= state_ >> 12;
      state_ ^= state_ << 25;
      state_ ^= state_ >> 27;
      w[i] = state_ * 0x2545F4914F6CDD1DULL;
    }
    return o;
  }
  EnvSpec s_;
  std::uint64_t state_ = 1;
  int steps_ = 0;
  bool done_ = true;
  bool single_ = false;
};

class RepeatWrapper final : public Env {  // envs.cpp:140-164
 public:
  RepeatWrapper(std::unique_ptr<Env> in, int k) : in_(std::move(in)), k_(k) {}
  Observation reset(std::uint64_t seed) override { return in_->reset(seed); }
  StepResult step(int a) override {
    StepResult out;
    for (int i = 0; i < k_; ++i) {
      StepResult r = in_->step(a);
      out.reward += r.reward;
      out.observation = std::move(r.observation);
      out.terminal = r.terminal;
      if (out.terminal) break;
    }
    return out;
  }
  int action_count() const override { return in_->action_count(); }
  bool frames() const override { return in_->frames(); }
  ga3c_net_spec input() const override { return in_->input(); }
  void set_single_frame(bool on) override { in_->set_single_frame(on); }

 private:
  std::unique_ptr<Env> in_;
  int k_;
};

}  // namespace

void validate(const EnvSpec& s) {
  if (s.action_repeat < 1) throw std::invalid_argument("EnvSpec: action_repeat must be >= 1");
  switch (s.kind) {
    case EnvKind::ContextualBandit:
      if (s.n_contexts < 1) throw std::invalid_argument("EnvSpec: n_contexts must be >= 1");
      if (s.n_actions < 2) throw std::invalid_argument("EnvSpec: n_actions must be >= 2");
      break;
    case EnvKind::Catch:
      if (s.grid_size < 2) throw std::invalid_argument("EnvSpec: grid_size must be >= 2");
      break;
    case EnvKind::DelayLab:
      if (s.step_delay_us < 0 || s.episode_len < 1) throw std::invalid_argument("EnvSpec: bad delay lab");
      break;
    case EnvKind::FrameCatch:
      if (s.grid_size < 2 || 84 % s.grid_size != 0 || s.n_actions < 3)
        throw std::invalid_argument("EnvSpec: frame catch needs grid_size | 84 and >= 3 actions");
      break;
    case EnvKind::Frames:
      if (s.step_delay_us < 0 || s.episode_len < 1 || s.n_actions < 2)
        throw std::invalid_argument("EnvSpec: bad frames env");
      break;
  }
}

std::unique_ptr<Env> make_env(const EnvSpec& s) {
  validate(s);
  std::unique_ptr<Env> e;
  switch (s.kind) {
    case EnvKind::ContextualBandit: e = std::make_unique<BanditEnv>(s); break;
    case EnvKind::Catch: e = std::make_unique<CatchEnv>(s); break;
    case EnvKind::DelayLab: e = std::make_unique<DelayLabEnv>(s); break;
    case EnvKind::FrameCatch: e = std::make_unique<FrameCatchEnv>(s); break;
    case EnvKind::Frames: e = std::make_unique<FramesEnv>(s); break;
  }
  if (s.action_repeat > 1) e = std::make_unique<RepeatWrapper>(std::move(e), s.action_repeat);
  return e;
}

// ---------------------------------------------------------------- knobs
void validate(const KnobConfig& k) {  // knobs.hpp:21-29
  if (k.n_agents < 1) throw std::invalid_argument("KnobConfig: n_agents must be >= 1");
  if (k.n_predictors < 1) throw std::invalid_argument("KnobConfig: n_predictors must be >= 1");
  if (k.n_trainers < 1) throw std::invalid_argument("KnobConfig: n_trainers must be >= 1");
  if (k.pred_batch_max < 1) throw std::invalid_argument("KnobConfig: pred_batch_max must be >= 1");
  if (k.min_train_batch < 1) throw std::invalid_argument("KnobConfig: min_train_batch must be >= 1");
  if (k.train_queue_cap < 1) throw std::invalid_argument("KnobConfig: train_queue_cap must be >= 1");
  if (k.pred_queue_cap < 0) throw std::invalid_argument("KnobConfig: pred_queue_cap must be >= 0");
}

// ------------------------------------------------------------- annealer
AnnealState make_anneal_state(const KnobConfig& initial, double epoch_length_s, std::uint64_t seed,
                              const Limits& limits, bool tune_batches) {  // annealer.cpp:9-26
  validate(initial);
  if (!(epoch_length_s > 0.0)) throw std::invalid_argument("annealer: epoch length must be positive");
  if (limits.max_agents < 1 || limits.max_predictors < 1 || limits.max_trainers < 1)
    throw std::invalid_argument("annealer: limits must be >= 1");
  if (initial.n_agents > limits.max_agents || initial.n_predictors > limits.max_predictors ||
      initial.n_trainers > limits.max_trainers)
    throw std::invalid_argument("annealer: initial config exceeds limits");
  AnnealState st;
  st.current = initial;
  st.epoch_length_s = epoch_length_s;
  st.limits = limits;
  st.tune_batches = tune_batches;
  st.rng.seed(mix64(seed));
  return st;
}

// annealer.cpp:28-53: one knob, +-1, redrawn until legal.  With tune_batches
// the two batch-geometry knobs join the draw and move by a factor of two in
// [1, 1024] (extension; off by default).
KnobConfig propose(AnnealState& s) {
  const int n_knobs = s.tune_batches ? 5 : 3;
  for (;;) {
    KnobConfig c = s.current;
    const int knob = static_cast<int>(next_uniform(s.rng) * n_knobs);
    const int delta = next_uniform(s.rng) < 0.5 ? -1 : 1;
    int* field = nullptr;
    int limit = 0;
    switch (knob) {
      case 0: field = &c.n_agents; limit = s.limits.max_agents; break;
      case 1: field = &c.n_predictors; limit = s.limits.max_predictors; break;
      case 2: field = &c.n_trainers; limit = s.limits.max_trainers; break;
      case 3: field = &c.pred_batch_max; limit = 1024; break;
      default: field = &c.min_train_batch; limit = 1024; break;
    }
    if (knob >= 3)
      *field = delta > 0 ? *field * 2 : *field / 2;
    else
      *field += delta;
    if (*field >= 1 && *field <= limit && !(c == s.current)) return c;
  }
}

bool decide(AnnealState& s, const KnobConfig& cand, double measured_tps) {
  HistoryEntry e{cand, measured_tps, false};
  if (measured_tps > s.baseline_tps) {
    s.current = cand;
    s.baseline_tps = measured_tps;
    e.accepted = true;
  } else {
    s.baseline_tps *= (1.0 - s.baseline_decay);
  }
  s.history.push_back(e);
  return e.accepted;
}

}  // namespace ga3c::host
