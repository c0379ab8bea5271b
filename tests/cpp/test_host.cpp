// test_host.cpp -- CPU unit tests of the host engine pieces that need no GPU:
// queues (test_channel.cpp), annealer (test_annealer.cpp), environments
// (test_envs.cpp) and the seed / sampling helpers (util.hpp).  Built and run
// by tests/test_host_cpp.py with g++ against csrc/host/envs.cpp.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <set>
#include <stdexcept>
#include <thread>
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
#define CHECK_THROWS(expr)                                                 \
  do {                                                                     \
    bool threw_ = false;                                                   \
    try {                                                                  \
      expr;                                                                \
    } catch (const std::exception&) {                                      \
      threw_ = true;                                                       \
    }                                                                      \
    CHECK(threw_);                                                         \
  } while (0)

static void channel_fifo_and_capacity() {  // test_channel.cpp:12-40
  BoundedChannel<int> q(2);
  CHECK(q.push(1));
  CHECK(q.push(2));
  CHECK(q.size() == 2);
  CHECK(*q.pop() == 1);
  CHECK(*q.try_pop() == 2);
  CHECK(!q.try_pop().has_value());
  q.close();
  CHECK(!q.push(3));
  CHECK(!q.pop().has_value());
}

static void channel_stop_wakes_blocked_pop() {
  BoundedChannel<int> q(1);
  std::atomic<bool> stop{false};
  std::atomic<bool> returned{false};
  std::thread t([&] {
    auto v = q.pop(&stop);
    returned = !v.has_value();
  });
  std::this_thread::sleep_for(std::chrono::milliseconds(20));
  stop = true;
  q.wake_all();
  t.join();
  CHECK(returned.load());
}

static void channel_mpmc_exactly_once() {  // test_channel.cpp:93-120
  BoundedChannel<int> q(8);
  const int producers = 4, consumers = 4, per = 2000;
  std::vector<std::thread> ts;
  std::vector<std::vector<int>> got(consumers);
  for (int p = 0; p < producers; ++p)
    ts.emplace_back([&, p] {
      for (int i = 0; i < per; ++i) q.push(p * per + i);
    });
  for (int c = 0; c < consumers; ++c)
    ts.emplace_back([&, c] {
      while (auto v = q.pop()) got[c].push_back(*v);
    });
  for (int p = 0; p < producers; ++p) ts[p].join();
  q.close();
  for (int c = 0; c < consumers; ++c) ts[producers + c].join();
  std::set<int> all;
  std::size_t n = 0;
  for (auto& g : got) {
    n += g.size();
    all.insert(g.begin(), g.end());
  }
  CHECK(n == static_cast<std::size_t>(producers * per));
  CHECK(all.size() == static_cast<std::size_t>(producers * per));
}

static void response_slot_tickets() {  // test_channel.cpp:139-160
  ResponseSlot<int> s;
  std::atomic<bool> stop{false};
  const auto t1 = s.issue_ticket();
  const auto t2 = s.issue_ticket();
  s.put(t2, 22);
  s.put(t1, 11);  // stale: must not overwrite the newer value
  CHECK(*s.take(t2, stop) == 22);
  stop = true;
  CHECK(!s.take(t1, stop).has_value());
}

static void annealer_walk() {  // test_annealer.cpp:28-153
  KnobConfig k;
  k.n_agents = 2;
  k.n_predictors = 1;
  k.n_trainers = 1;
  Limits lim{4, 3, 3};
  auto st = make_anneal_state(k, 1.0, 42, lim);
  for (int i = 0; i < 2000; ++i) {
    const KnobConfig c = propose(st);
    int moved = (c.n_agents != st.current.n_agents) + (c.n_predictors != st.current.n_predictors) +
                (c.n_trainers != st.current.n_trainers);
    CHECK(moved == 1);
    CHECK(c.n_agents >= 1 && c.n_agents <= 4 && c.n_predictors >= 1 && c.n_predictors <= 3);
    CHECK(c.n_trainers >= 1 && c.n_trainers <= 3);
    CHECK(c.pred_batch_max == k.pred_batch_max && c.min_train_batch == k.min_train_batch);
    decide(st, c, static_cast<double>(i % 7));
  }
  auto s2 = make_anneal_state(k, 1.0, 1, lim);
  s2.baseline_tps = 10.0;
  CHECK(!decide(s2, k, 9.0));
  CHECK(std::abs(s2.baseline_tps - 9.9) < 1e-12);  // 1% decay per reject
  CHECK(decide(s2, k, 11.0));
  CHECK(s2.baseline_tps == 11.0);
  CHECK_THROWS(make_anneal_state(k, 0.0, 1, lim));
  k.n_agents = 9;
  CHECK_THROWS(make_anneal_state(k, 1.0, 1, lim));
  // batch-geometry extension: moves by factors of two inside [1, 1024]
  KnobConfig kb;
  auto sb = make_anneal_state(kb, 1.0, 7, Limits{}, true);
  bool batch_moved = false;
  for (int i = 0; i < 500; ++i) {
    const KnobConfig c = propose(sb);
    CHECK(c.pred_batch_max >= 1 && c.pred_batch_max <= 1024 && c.min_train_batch >= 1 && c.min_train_batch <= 1024);
    batch_moved |= c.pred_batch_max != kb.pred_batch_max || c.min_train_batch != kb.min_train_batch;
  }
  CHECK(batch_moved);
}

static void envs_dynamics() {  // test_envs.cpp
  EnvSpec cs;
  cs.kind = EnvKind::Catch;
  cs.grid_size = 5;
  auto c = make_env(cs);
  c->reset(3);
  int steps = 0;
  StepResult r;
  do {
    r = c->step(1);
    ++steps;
  } while (!r.terminal);
  CHECK(steps == 4);
  CHECK(r.reward == 1.0 || r.reward == -1.0);
  CHECK_THROWS(c->step(1));
  EnvSpec bs;
  auto b = make_env(bs);
  const auto o = b->reset(5);
  int ctx = 0;
  for (int i = 0; i < 4; ++i)
    if (o.f32[i] == 1.f) ctx = i;
  CHECK(b->step(ctx % 4).reward == 1.0);
  EnvSpec fs;
  fs.kind = EnvKind::FrameCatch;
  fs.grid_size = 7;
  fs.n_actions = 6;
  auto f = make_env(fs);
  const auto fo = f->reset(9);
  CHECK(fo.u8.size() == 84u * 84u * 4u);
  CHECK(f->frames());
  int lit = 0;
  for (std::size_t i = 3; i < fo.u8.size(); i += 4) lit += fo.u8[i] != 0;
  CHECK(lit == 2 * 12 * 12);  // ball + paddle cells in the newest frame
  EnvSpec xs;
  xs.kind = EnvKind::Frames;
  xs.step_delay_us = 0;
  xs.episode_len = 3;
  xs.n_actions = 6;
  auto x = make_env(xs);
  x->reset(1);
  x->step(0);
  x->step(0);
  CHECK(x->step(0).terminal);
  EnvSpec bad;
  bad.kind = EnvKind::FrameCatch;
  bad.grid_size = 5;  // 84 % 5 != 0
  CHECK_THROWS(make_env(bad));
  EnvSpec rep;
  rep.kind = EnvKind::Catch;
  rep.grid_size = 5;
  rep.action_repeat = 2;
  auto rr = make_env(rep);
  rr->reset(2);
  int n = 0;
  StepResult s;
  do {
    s = rr->step(1);
    ++n;
  } while (!s.terminal);
  CHECK(n == 2);
}

static void sampling_matches_util() {  // util.hpp:46-54
  std::mt19937_64 a(1234), b(1234);
  const double p[4] = {0.1, 0.2, 0.3, 0.4};
  int counts[4] = {0, 0, 0, 0};
  for (int i = 0; i < 40000; ++i) {
    const double u = next_uniform(b);
    double acc = 0.0;
    int want = 3;
    for (int k = 0; k < 4; ++k) {
      acc += p[k];
      if (u < acc) {
        want = k;
        break;
      }
    }
    const int got = sample_index(p, 4, a);
    CHECK(got == want);
    counts[got]++;
  }
  CHECK(std::abs(counts[3] / 40000.0 - 0.4) < 0.02);
  CHECK(argmax_index(p, 4) == 3);
  CHECK(derive_seed(1, {kSeedModelInit}) == derive_seed(1, {kSeedModelInit}));
  CHECK(derive_seed(1, {kSeedAgentRng, 0}) != derive_seed(1, {kSeedAgentRng, 1}));
}

int main() {
  channel_fifo_and_capacity();
  channel_stop_wakes_blocked_pop();
  channel_mpmc_exactly_once();
  response_slot_tickets();
  annealer_walk();
  envs_dynamics();
  sampling_matches_util();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
