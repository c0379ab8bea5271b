// test_engine_gpu.cpp -- the host engine's own predictor_loop and trainer
// pool against the device (libga3c_b200.so), restating the reference's
// direct predictor tests (/root/reference/proj/tests/test_pipeline.cpp:45-98)
// on ga3c::host::predictor_loop, plus its frame-store mode and the native
// trainer pool.  Built and run by tests/test_engine_gpu.py (-m gpu).
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "channel.hpp"
#include "ga3c_host.hpp"

using namespace ga3c::host;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                           \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(c)) {                                                            \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);             \
    }                                                                      \
  } while (0)

namespace {

std::vector<std::unique_ptr<ResponseSlot<PredictionResponse>>> make_slots(int n) {
  std::vector<std::unique_ptr<ResponseSlot<PredictionResponse>>> s;
  for (int i = 0; i < n; ++i) s.push_back(std::make_unique<ResponseSlot<PredictionResponse>>());
  return s;
}

ga3c_net_spec mlp(int in, std::vector<int> hidden, int actions) {
  ga3c_net_spec s{};
  s.in_h = s.in_w = 1;
  s.in_c = in;
  s.n_hidden = static_cast<int>(hidden.size());
  for (std::size_t i = 0; i < hidden.size(); ++i) s.hidden[i] = hidden[i];
  s.n_actions = actions;
  return s;
}

ga3c_hyper hyper() {
  ga3c_hyper h;
  ga3c_default_hyper(&h);
  return h;
}

Observation f32_state(std::vector<float> v) {
  Observation o;
  o.f32 = std::move(v);
  return o;
}

}  // namespace

// test_pipeline.cpp:45-78: everything queued is answered by ONE forward,
// whose output equals a direct batched forward of the same states bitwise.
static void predictor_answers_queue_with_one_forward() {
  const ga3c_net_spec spec = mlp(4, {8}, 3);
  SharedModel model(spec, hyper(), 0, 77);
  auto slots = make_slots(7);
  BoundedChannel<PredictionRequest> q(16);
  PredictorMetrics metrics;
  std::atomic<bool> stop{false};
  std::vector<float> states;
  std::vector<std::uint64_t> tickets;
  for (int i = 0; i < 7; ++i) {
    std::vector<float> s{0.1f * i, -0.2f * i, 0.3f, 1.0f};
    states.insert(states.end(), s.begin(), s.end());
    const auto t = slots[i]->issue_ticket();
    tickets.push_back(t);
    CHECK(q.push(PredictionRequest{i, t, f32_state(s)}));
  }
  q.close();  // drained, then the loop exits on the closed channel
  int st = 0;
  ga3c_ctx* ctx = ga3c_ctx_create(model.handle(), 32, &st);
  CHECK(ctx != nullptr);
  predictor_loop(q, slots, model, ctx, 32, metrics, stop);
  CHECK(metrics.predictions.load() == 7);
  CHECK(metrics.batches.load() == 1);  // a single batch served all requests

  std::vector<double> pi(7 * 3), v(7);
  std::uint64_t ver = 99;
  CHECK(ga3c_forward64_f32(ctx, -1, states.data(), 7, pi.data(), v.data(), &ver) == GA3C_OK);
  for (int i = 0; i < 7; ++i) {
    auto resp = slots[i]->take(tickets[i], stop);
    CHECK(resp.has_value());
    if (!resp) continue;
    CHECK(resp->policy.size() == 3);
    CHECK(std::memcmp(resp->policy.data(), pi.data() + 3 * i, 3 * sizeof(double)) == 0);
    CHECK(resp->value == v[i]);
    CHECK(resp->model_version == 0 && ver == 0);
  }
  ga3c_ctx_destroy(ctx);
}

// test_pipeline.cpp:80-98: batches are capped at pred_batch_max.
static void prediction_batches_capped() {
  const ga3c_net_spec spec = mlp(4, {}, 2);
  SharedModel model(spec, hyper(), 0, 3);
  auto slots = make_slots(10);
  BoundedChannel<PredictionRequest> q(16);
  PredictorMetrics metrics;
  std::atomic<bool> stop{false};
  for (int i = 0; i < 10; ++i) CHECK(q.push(PredictionRequest{i, slots[i]->issue_ticket(), f32_state({1, 0, 0, 0})}));
  q.close();
  int st = 0;
  ga3c_ctx* ctx = ga3c_ctx_create(model.handle(), 4, &st);
  predictor_loop(q, slots, model, ctx, 4, metrics, stop);
  CHECK(metrics.predictions.load() == 10);
  CHECK(metrics.batches.load() == 3);  // 4, 4, 2
  ga3c_ctx_destroy(ctx);
}

// Frame-store mode: requests carry the newest 84x84 frame; the stacked state
// the device forwards is [oldest .. newest] with an episode start repeated
// four times, and the response names the slot that holds it.
static void predictor_frame_store_mode() {
  ga3c_net_spec spec{};
  spec.in_h = spec.in_w = 84;
  spec.in_c = 4;
  spec.n_conv = 2;
  spec.conv_out[0] = 16, spec.conv_k[0] = 8, spec.conv_stride[0] = 4;
  spec.conv_out[1] = 32, spec.conv_k[1] = 4, spec.conv_stride[1] = 2;
  spec.n_hidden = 1;
  spec.hidden[0] = 256;
  spec.n_actions = 6;
  SharedModel model(spec, hyper(), 0, 5);
  int st = 0;
  ga3c_frames* store = ga3c_frames_create(model.handle(), 3, 8, &st);
  CHECK(store != nullptr);
  ga3c_ctx* ctx = ga3c_ctx_create(model.handle(), 8, &st);
  const int px = 84 * 84;
  auto frame = [&](int agent, int step) {
    Observation o;
    o.u8.resize(px);
    for (int p = 0; p < px; ++p) o.u8[p] = static_cast<std::uint8_t>((p * 7 + agent * 31 + step * 13) & 0xff);
    return o;
  };
  auto slots = make_slots(3);
  PredictorMetrics metrics;
  std::atomic<bool> stop{false};
  std::vector<int> got_slot(3, -1);
  for (int step = 0; step < 3; ++step) {
    BoundedChannel<PredictionRequest> q(8);
    std::vector<std::uint64_t> tk(3);
    for (int a = 0; a < 3; ++a) {
      tk[a] = slots[a]->issue_ticket();
      CHECK(q.push(PredictionRequest{a, tk[a], frame(a, step), step == 0}));
    }
    q.close();
    predictor_loop(q, slots, model, ctx, 8, metrics, stop, store);
    for (int a = 0; a < 3; ++a) {
      auto r = slots[a]->take(tk[a], stop);
      CHECK(r.has_value() && r->state_slot >= 0);
      if (r) got_slot[a] = r->state_slot;
    }
  }
  // after 3 pushes agent a's stack is [f0, f0, f1, f2] (reset at step 0)
  for (int a = 0; a < 3; ++a) {
    std::vector<std::uint8_t> s(4 * px);
    CHECK(ga3c_frames_read(store, a, got_slot[a], s.data()) == GA3C_OK);
    const Observation f0 = frame(a, 0), f1 = frame(a, 1), f2 = frame(a, 2);
    bool ok = true;
    for (int p = 0; p < px && ok; ++p)
      ok = s[4 * p] == f0.u8[p] && s[4 * p + 1] == f0.u8[p] && s[4 * p + 2] == f1.u8[p] && s[4 * p + 3] == f2.u8[p];
    CHECK(ok);
  }
  CHECK(metrics.batches.load() == 3 && metrics.predictions.load() == 9);
  ga3c_ctx_destroy(ctx);
  ga3c_frames_destroy(store);
}

// The native trainer pool: every submitted batch is applied, in FIFO order
// with one thread the result equals the same train_frames + apply sequence
// run directly, bitwise.
static void trainer_pool_matches_direct_calls() {
  ga3c_net_spec spec{};
  spec.in_h = spec.in_w = 84;
  spec.in_c = 4;
  spec.n_conv = 2;
  spec.conv_out[0] = 16, spec.conv_k[0] = 8, spec.conv_stride[0] = 4;
  spec.conv_out[1] = 32, spec.conv_k[1] = 4, spec.conv_stride[1] = 2;
  spec.n_hidden = 1;
  spec.hidden[0] = 256;
  spec.n_actions = 6;
  const int NA = 8, T = 5, px = 84 * 84;
  auto run = [&](bool pooled) {
    SharedModel model(spec, hyper(), 0, 11);
    int st = 0;
    ga3c_frames* store = ga3c_frames_create(model.handle(), NA, 2 * T, &st);
    ga3c_ctx* pc = ga3c_ctx_create(model.handle(), NA, &st);
    std::vector<std::uint8_t> newf(NA * px);
    std::vector<std::int32_t> agents(NA), slots(NA * T);
    for (int a = 0; a < NA; ++a) agents[a] = a;
    std::vector<double> pi(NA * 6), v(NA);
    for (int t = 0; t < T; ++t) {
      for (int i = 0; i < NA * px; ++i) newf[i] = static_cast<std::uint8_t>((i * 3 + t * 101) & 0xff);
      std::vector<std::int32_t> sl(NA);
      CHECK(ga3c_predict_frames64(pc, -1, store, newf.data(), agents.data(), nullptr, NA, sl.data(), pi.data(),
                                  v.data(), nullptr) == GA3C_OK);
      for (int a = 0; a < NA; ++a) slots[a * T + t] = sl[a];
    }
    // two updates of 4 agents x T steps
    ga3c_trainer_pool* pool = pooled ? ga3c_trainer_pool_create(model.handle(), store, 1, 64, 0, 4, &st) : nullptr;
    ga3c_ctx* tc = pooled ? nullptr : ga3c_ctx_create(model.handle(), 64, &st);
    for (int u = 0; u < 2; ++u) {
      std::vector<std::int32_t> ag, sl, act, off{0};
      std::vector<double> rew, boot;
      std::vector<std::uint8_t> term;
      for (int a = 4 * u; a < 4 * u + 4; ++a) {
        for (int t = 0; t < T; ++t) {
          ag.push_back(a);
          sl.push_back(slots[a * T + t]);
          act.push_back((a + t) % 6);
          rew.push_back(0.25 * ((a + 2 * t) % 5) - 0.5);
        }
        off.push_back(static_cast<std::int32_t>(ag.size()));
        term.push_back(a % 3 == 0);
        boot.push_back(0.1 * a);
      }
      const int B = static_cast<int>(ag.size()), n = static_cast<int>(term.size());
      if (pooled) {
        CHECK(ga3c_trainer_pool_submit(pool, ag.data(), sl.data(), B, act.data(), rew.data(), off.data(), n,
                                       term.data(), boot.data(), 0.99) == GA3C_OK);
      } else {
        CHECK(ga3c_train_frames(tc, -1, store, ag.data(), sl.data(), B, act.data(), rew.data(), off.data(), n,
                                term.data(), boot.data(), 0.99, 1, nullptr, nullptr) == GA3C_OK);
        int applied = 0;
        CHECK(ga3c_apply_rmsprop(tc, nullptr, &applied, nullptr) == GA3C_OK && applied == 1);
      }
    }
    if (pooled) {
      long long upd = 0, rej = 0;
      CHECK(ga3c_trainer_pool_wait(pool, &upd, &rej) == GA3C_OK);
      CHECK(upd == 2 && rej == 0);
      ga3c_trainer_pool_destroy(pool);
    } else {
      ga3c_ctx_destroy(tc);
    }
    std::vector<float> th = model.read_theta();
    CHECK(model.version() == 2);
    ga3c_ctx_destroy(pc);
    ga3c_frames_destroy(store);
    return th;
  };
  const auto a = run(true), b = run(false);
  CHECK(a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0);
}

int main() {
  predictor_answers_queue_with_one_forward();
  prediction_batches_capped();
  predictor_frame_store_mode();
  trainer_pool_matches_direct_calls();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
