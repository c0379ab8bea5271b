// test_dropin.cpp -- the reference ENGINE running on the B200 library.
//
// This driver is linked against the reference's own, unmodified engine
// sources (/root/reference/proj/src/{pipeline,reference,envs,metrics,
// annealer}.cpp), compiled by oracle/Makefile target `dropin` with this
// repository's include/ ahead of the reference's, so that the reference's
// `#include "qac/nnet.hpp"` / `"qac/returns.hpp"` resolve to the shims in
// include/qac/ and every nnet:: / returns:: call the engine makes runs on
// libga3c_b200.so.  The same driver is also linked against the reference's
// CPU nnet.cpp / returns.cpp (binary test_dropin_cpu) so a test can compare
// the two trajectories.
//
// Modes
//   test_dropin_<impl> run
//       the reference's pipeline tests (tests/test_pipeline.cpp:45-320),
//       restated as checks on whichever nnet this binary links;
//   test_dropin_<impl> traj SEED UPDATES OUT
//       reference::train_sync (reference.cpp:25-157) on catch_grid(4) with a
//       {16} trunk; writes the post-update theta trajectory and the episode
//       scores to OUT (int64 n, int64 P, n*P doubles, int64 k, k doubles).
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "qac/channel.hpp"
#include "qac/cli.hpp"
#include "qac/pipeline.hpp"
#include "qac/reference.hpp"

namespace {

int g_checks = 0, g_failures = 0;

void expect(bool ok, const char* what, int line) {
  ++g_checks;
  if (!ok) {
    ++g_failures;
    std::printf("  FAILED line %d: %s\n", line, what);
  }
}
#define EXPECT(c) expect((c), #c, __LINE__)

template <typename F>
void expect_invalid(F&& f, const char* what, int line) {
  bool thrown = false;
  try {
    f();
  } catch (const std::invalid_argument&) {
    thrown = true;
  } catch (...) {
  }
  expect(thrown, what, line);
}
#define EXPECT_INVALID(expr) expect_invalid([&] { (void)(expr); }, #expr " throws invalid_argument", __LINE__)

void run_case(const char* name, const std::function<void()>& body) {
  const int before = g_failures;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_failures;
    std::printf("  FAILED: exception %s\n", e.what());
  }
  std::printf("%s %s\n", g_failures == before ? "[ok]  " : "[FAIL]", name);
}

using namespace qac;
using pipeline::PipelineOptions;
using pipeline::PredictionRequest;
using pipeline::PredictionResponse;
using Slots = std::vector<std::unique_ptr<ResponseSlot<PredictionResponse>>>;

Slots response_slots(int n) {
  Slots s;
  for (int i = 0; i < n; ++i) s.push_back(std::make_unique<ResponseSlot<PredictionResponse>>());
  return s;
}

// test_pipeline.cpp:21-34: the 1/1/1 lock-step shape with min_train_batch 1
PipelineOptions lockstep(const envs::EnvSpec& env, std::int64_t updates, std::uint64_t seed) {
  PipelineOptions o;
  o.env = env;
  o.net = cli::net_for_env(env, {16});
  o.knobs.n_agents = o.knobs.n_predictors = o.knobs.n_trainers = 1;
  o.knobs.min_train_batch = 1;
  o.stop.max_updates = updates;
  o.seed = seed;
  o.sync_after_submit = true;
  return o;
}

// test_pipeline.cpp:45-78
void predictor_single_forward() {
  const nnet::NetworkSpec spec{4, {8}, 3};
  pipeline::SharedModel model(nnet::init_model(spec, 77), nnet::init_rms(spec));
  Slots slots = response_slots(7);
  BoundedChannel<PredictionRequest> q(16);
  metrics::MetricsCollector mc;
  std::atomic<bool> stop{false};
  std::vector<std::vector<double>> states;
  std::vector<std::uint64_t> tickets;
  for (int i = 0; i < 7; ++i) {
    states.push_back({0.1 * i, -0.2 * i, 0.3, 1.0});
    tickets.push_back(slots[i]->issue_ticket());
    EXPECT(q.push(PredictionRequest{i, tickets.back(), states.back()}));
  }
  q.close();
  pipeline::predictor_loop(q, slots, model, spec, 32, mc, stop);
  EXPECT(mc.predictions_total() == 7);
  EXPECT(mc.snapshot(0, 1, 0, 1.0).pred_batch_mean == 7.0);
  const auto want = nnet::forward(*model.snapshot(), spec, states);
  for (int i = 0; i < 7; ++i) {
    const auto r = slots[i]->take(tickets[i], stop);
    EXPECT(r.has_value());
    if (!r) continue;
    EXPECT(r->policy == want.policies[i]);  // bitwise: same device path, same batch
    EXPECT(r->value == want.values[i]);
    EXPECT(r->model_version == 0);
    double sum = 0.0;
    for (double p : r->policy) sum += p;
    EXPECT(std::fabs(sum - 1.0) < 1e-12);  // fp64 softmax across the ABI
  }
}

// test_pipeline.cpp:80-98
void predictor_batch_cap() {
  const nnet::NetworkSpec spec{4, {}, 2};
  pipeline::SharedModel model(nnet::init_model(spec, 3), nnet::init_rms(spec));
  Slots slots = response_slots(10);
  BoundedChannel<PredictionRequest> q(16);
  metrics::MetricsCollector mc;
  std::atomic<bool> stop{false};
  for (int i = 0; i < 10; ++i)
    EXPECT(q.push(PredictionRequest{i, slots[i]->issue_ticket(), {1.0, 0.0, 0.0, 0.0}}));
  q.close();
  pipeline::predictor_loop(q, slots, model, spec, 4, mc, stop);
  EXPECT(mc.predictions_total() == 10);
  EXPECT(mc.snapshot(0, 1, 0, 1.0).pred_batch_mean == 10.0 / 3.0);  // 4 + 4 + 2
}

// test_pipeline.cpp:100-121
void shared_model_serial_apply() {
  const nnet::NetworkSpec spec{2, {}, 2};
  const nnet::Hyperparams hp;
  pipeline::SharedModel model(nnet::init_model(spec, 9), nnet::init_rms(spec));
  const auto before = model.snapshot();
  EXPECT(before->version == 0);
  nnet::GradientPacket g;
  g.dtheta.assign(nnet::param_count(spec), 0.5);
  g.batch_size = 1;
  const auto on = model.apply(g, hp);
  EXPECT(on.has_value() && *on == 0);
  EXPECT(model.version() == 1);
  EXPECT(before->version == 0);
  EXPECT(before->theta != model.snapshot()->theta);
  g.dtheta[0] = std::nan("");
  EXPECT(!model.apply(g, hp).has_value());
  EXPECT(model.version() == 1);
}

// test_pipeline.cpp:123-148
void lockstep_matches_serial() {
  for (const std::uint64_t seed : {7u, 19u}) {
    auto o = lockstep(envs::catch_grid(4), 120, seed);
    o.capture_trajectory = true;
    reference::SyncConfig sc;
    sc.env = o.env;
    sc.net = o.net;
    sc.hyper = o.hyper;
    sc.max_updates = 120;
    sc.seed = seed;
    sc.capture_trajectory = true;
    const auto piped = pipeline::run(o);
    const auto serial = reference::train_sync(sc);
    EXPECT(piped.total_updates == 120);
    EXPECT(piped.theta_trajectory.size() == 120 && serial.theta_trajectory.size() == 120);
    bool same = piped.theta_trajectory.size() == serial.theta_trajectory.size();
    for (std::size_t i = 0; same && i < piped.theta_trajectory.size(); ++i)
      same = piped.theta_trajectory[i] == serial.theta_trajectory[i];
    EXPECT(same);
    EXPECT(piped.final_model.theta == serial.final_model.theta);
    EXPECT(piped.episode_scores == serial.episode_scores);
    EXPECT(piped.mean_lag == 0.0);
  }
}

// test_pipeline.cpp:150-158
void greedy_reproducible() {
  auto o = lockstep(envs::catch_grid(4), 40, 33);
  o.greedy = true;
  const auto a = pipeline::run(o);
  const auto b = pipeline::run(o);
  EXPECT(a.final_model.theta == b.final_model.theta);
  EXPECT(a.total_episodes == b.total_episodes);
  EXPECT(a.episode_scores == b.episode_scores);
}

// test_pipeline.cpp:160-176
void conservation() {
  PipelineOptions o;
  o.env = envs::catch_grid(5);
  o.net = cli::net_for_env(o.env, {16});
  o.knobs.n_agents = 3;
  o.knobs.n_predictors = 2;
  o.knobs.n_trainers = 2;
  o.knobs.min_train_batch = 8;
  o.stop.max_updates = 60;
  o.seed = 123;
  const auto r = pipeline::run(o);
  EXPECT(r.total_updates == 60);
  EXPECT(r.experiences_produced == r.experiences_trained + r.experiences_left_queued + r.experiences_dropped);
  EXPECT(r.experiences_trained >= 60 * 8);
  EXPECT(r.total_episodes == static_cast<std::int64_t>(r.episode_scores.size()));
}

// test_pipeline.cpp:178-196
void coalescing() {
  PipelineOptions o;
  o.env = envs::bandit();
  o.net = cli::net_for_env(o.env, {8});
  o.knobs.n_agents = 2;
  o.knobs.min_train_batch = 7;
  o.stop.max_updates = 25;
  o.seed = 5;
  const auto r = pipeline::run(o);
  EXPECT(r.total_updates == 25);
  EXPECT(r.experiences_trained == 25 * 7);
  EXPECT(r.experiences_produced == r.experiences_trained + r.experiences_left_queued + r.experiences_dropped);
}

// test_pipeline.cpp:198-220
void staleness_recorded() {
  PipelineOptions o;
  o.env = envs::catch_grid(5);
  o.net = cli::net_for_env(o.env, {16});
  o.knobs.n_agents = 4;
  o.knobs.min_train_batch = 1;
  o.stop.max_updates = 300;
  o.seed = 99;
  const auto r = pipeline::run(o);
  EXPECT(r.total_updates == 300);
  EXPECT(r.mean_lag >= 0.0 && std::isfinite(r.mean_lag));
  EXPECT(!r.frames.empty());
  if (!r.frames.empty()) {
    EXPECT(r.frames.back().n_a == 4);
    EXPECT(r.frames.back().updates_total == 300);
  }
}

// test_pipeline.cpp:222-246
void stop_conditions() {
  PipelineOptions o;
  o.env = envs::bandit(2, 2);
  o.net = cli::net_for_env(o.env, {8});
  o.stop = {};
  o.stop.max_seconds = 0.3;
  o.seed = 3;
  const auto r = pipeline::run(o);
  EXPECT(r.wall_time_s >= 0.3 && r.wall_time_s < 30.0);
  EXPECT(r.total_updates > 0);
  PipelineOptions o2 = o;
  o2.stop = {};
  o2.stop.target_score = 0.9;
  o2.hyper.eta = 0.01;
  const auto r2 = pipeline::run(o2);
  EXPECT(r2.final_rolling_score >= 0.9);
  EXPECT(r2.total_episodes >= 30);
}

// test_pipeline.cpp:248-280
void annealing_limits() {
  PipelineOptions o;
  o.env = envs::bandit();
  o.net = cli::net_for_env(o.env, {8});
  o.knobs.n_agents = 2;
  o.anneal = true;
  o.epoch_s = 0.2;
  o.limits = {4, 3, 3};
  o.stop = {};
  o.stop.max_seconds = 2.0;
  o.seed = 17;
  const auto r = pipeline::run(o);
  EXPECT(r.anneal_history.size() >= 2);
  for (const auto& h : r.anneal_history) {
    EXPECT(h.knobs.n_agents >= 1 && h.knobs.n_agents <= 4);
    EXPECT(h.knobs.n_predictors >= 1 && h.knobs.n_predictors <= 3);
    EXPECT(h.knobs.n_trainers >= 1 && h.knobs.n_trainers <= 3);
    EXPECT(h.measured_tps >= 0.0);
  }
  EXPECT(r.final_knobs.min_train_batch == o.knobs.min_train_batch);
  EXPECT(r.final_knobs.pred_batch_max == o.knobs.pred_batch_max);
}

// test_pipeline.cpp:282-320
void option_validation() {
  const auto good = lockstep(envs::bandit(), 5, 1);
  auto o = good;
  o.stop = {};
  EXPECT_INVALID(pipeline::run(o));
  o = good;
  o.knobs.n_agents = 2;
  EXPECT_INVALID(pipeline::run(o));
  o = good;
  o.knobs.min_train_batch = 2;
  EXPECT_INVALID(pipeline::run(o));
  o = good;
  o.net.input_dim += 1;
  EXPECT_INVALID(pipeline::run(o));
  o = good;
  o.net.n_actions += 1;
  EXPECT_INVALID(pipeline::run(o));
  o = good;
  o.knobs.n_predictors = 0;
  EXPECT_INVALID(pipeline::run(o));
}

int write_trajectory(std::uint64_t seed, std::int64_t updates, const char* path) {
  reference::SyncConfig sc;
  sc.env = envs::catch_grid(4);
  sc.net = cli::net_for_env(sc.env, {16});
  sc.max_updates = updates;
  sc.seed = seed;
  sc.capture_trajectory = true;
  const auto r = reference::train_sync(sc);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return 2;
  const std::int64_t n = static_cast<std::int64_t>(r.theta_trajectory.size());
  const std::int64_t P = n ? static_cast<std::int64_t>(r.theta_trajectory[0].size()) : 0;
  std::fwrite(&n, sizeof n, 1, f);
  std::fwrite(&P, sizeof P, 1, f);
  for (const auto& t : r.theta_trajectory) std::fwrite(t.data(), sizeof(double), t.size(), f);
  const std::int64_t k = static_cast<std::int64_t>(r.episode_scores.size());
  std::fwrite(&k, sizeof k, 1, f);
  std::fwrite(r.episode_scores.data(), sizeof(double), r.episode_scores.size(), f);
  std::fclose(f);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "run";
  if (mode == "traj" && argc == 5)
    return write_trajectory(std::strtoull(argv[2], nullptr, 10), std::strtoll(argv[3], nullptr, 10), argv[4]);
  if (mode != "run") {
    std::fprintf(stderr, "usage: %s run | traj SEED UPDATES OUT\n", argv[0]);
    return 2;
  }
  run_case("predictor answers everything queued with one forward", predictor_single_forward);
  run_case("prediction batches are capped at pred_batch_max", predictor_batch_cap);
  run_case("shared model applies serially, snapshots immutable", shared_model_serial_apply);
  run_case("lockstep pipeline reproduces train_sync bit for bit", lockstep_matches_serial);
  run_case("greedy lockstep runs are reproducible", greedy_reproducible);
  run_case("every produced experience is accounted for", conservation);
  run_case("trainers coalesce submissions up to the batch floor", coalescing);
  run_case("a free-running pipeline records its staleness", staleness_recorded);
  run_case("stop conditions: wall clock and target score", stop_conditions);
  run_case("annealing stays within limits", annealing_limits);
  run_case("pipeline option validation", option_validation);
  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures ? 1 : 0;
}
