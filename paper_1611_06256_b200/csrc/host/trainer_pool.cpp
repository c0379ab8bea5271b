// trainer_pool.cpp -- GA3C's TrainingQueue + trainer threads
// (/root/reference/proj/src/pipeline.cpp:241-306) as a standalone component
// of the C ABI (include/ga3c.h "trainer pool"), for callers that run their
// own agents / predictors (the bench's e2e leg, a Python or Go host) and
// want the trainers native: submit() copies one segment batch (agents x
// frame-store slots, actions, rewards, segment table) into a bounded FIFO
// and returns; each of n_threads C++ trainers owns a ga3c_ctx, pops a batch,
// runs ga3c_train_frames (device returns + loss/backward on the states kept
// in the frame store) on the latest snapshot and ga3c_apply_rmsprop
// (out-of-place RMSProp, published at once).  No Python, no GIL on the
// training path.  The trainer contexts run one stream-priority level below
// the default (ga3c_ctx_set_priority), so the callers' predictions, which
// the agents wait on, are scheduled ahead of queued training kernels.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ga3c.h"

namespace {

struct Job {
  std::vector<std::int32_t> agents, slots, actions, seg_off;
  std::vector<double> rewards, bootstrap;
  std::vector<std::uint8_t> terminal;
  double gamma = 0.0;
};

}  // namespace

struct ga3c_trainer_pool {
  ga3c_model* m = nullptr;
  ga3c_frames* f = nullptr;
  int cap = 0;
  std::vector<std::thread> threads;
  std::vector<ga3c_ctx*> ctxs;
  std::mutex mu;
  std::condition_variable not_empty, not_full, idle;
  std::deque<Job> q;
  int busy = 0;
  bool closing = false;
  long long updates = 0, rejected = 0;
  int error = GA3C_OK;
  std::string error_msg;

  void worker(ga3c_ctx* c) {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        not_empty.wait(lk, [&] { return closing || !q.empty(); });
        if (q.empty()) return;  // closing and drained
        j = std::move(q.front());
        q.pop_front();
        ++busy;
      }
      not_full.notify_one();
      int st = ga3c_train_frames(c, -1, f, j.agents.data(), j.slots.data(), static_cast<int>(j.agents.size()),
                                 j.actions.data(), j.rewards.data(), j.seg_off.data(),
                                 static_cast<int>(j.terminal.size()), j.terminal.data(), j.bootstrap.data(),
                                 j.gamma, 1, nullptr, nullptr);
      int applied = 0;
      if (st == GA3C_OK) {
        st = ga3c_apply_rmsprop(c, nullptr, &applied, nullptr);
        if (st == GA3C_NOT_APPLIED) st = GA3C_OK;  // rejected step (nnet.cpp:299-301), counted below
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        --busy;
        if (st != GA3C_OK && error == GA3C_OK) {
          error = st;
          error_msg = ga3c_model_last_error(m);
        }
        if (st == GA3C_OK) (applied ? updates : rejected) += 1;
        if (q.empty() && busy == 0) idle.notify_all();
      }
    }
  }
};

extern "C" {

ga3c_trainer_pool* ga3c_trainer_pool_create(ga3c_model* m, ga3c_frames* f, int n_threads, int max_batch, int sms,
                                            int queue_cap, int* status) {
  auto fail = [&](int st) -> ga3c_trainer_pool* {
    if (status) *status = st;
    return nullptr;
  };
  if (!m || !f || n_threads < 1 || max_batch < 1 || queue_cap < 1 || sms < 0) return fail(GA3C_INVALID_ARGUMENT);
  auto* p = new ga3c_trainer_pool();
  p->m = m;
  p->f = f;
  p->cap = queue_cap;
  for (int i = 0; i < n_threads; ++i) {
    int st = 0;
    ga3c_ctx* c = ga3c_ctx_create(m, max_batch, &st);
    if (!c) {
      for (auto* x : p->ctxs) ga3c_ctx_destroy(x);
      delete p;
      return fail(st ? st : GA3C_CUDA_ERROR);
    }
    ga3c_ctx_set_sm_budget(c, sms);
    // one level below the callers' predictor contexts (DNN A e2e, two runs
    // each: level 0 835K / 869K, level 1 925K / 914K, level 3 921K / 856K)
    p->ctxs.push_back(c);
    const int pst = ga3c_ctx_set_priority(c, 1);
    if (pst != GA3C_OK) {
      for (auto* x : p->ctxs) ga3c_ctx_destroy(x);
      delete p;
      return fail(pst);
    }
  }
  for (auto* c : p->ctxs) p->threads.emplace_back([p, c] { p->worker(c); });
  if (status) *status = GA3C_OK;
  return p;
}

int ga3c_trainer_pool_submit(ga3c_trainer_pool* p, const int32_t* agents, const int32_t* state_slots, int B,
                             const int32_t* actions, const double* rewards, const int32_t* seg_offsets, int n_seg,
                             const uint8_t* terminal, const double* bootstrap, double gamma) {
  if (!p || B < 1 || n_seg < 1 || !agents || !state_slots || !actions || !rewards || !seg_offsets || !terminal ||
      !bootstrap)
    return GA3C_INVALID_ARGUMENT;
  if (seg_offsets[0] != 0 || seg_offsets[n_seg] != B) return GA3C_INVALID_ARGUMENT;
  Job j;
  j.agents.assign(agents, agents + B);
  j.slots.assign(state_slots, state_slots + B);
  j.actions.assign(actions, actions + B);
  j.rewards.assign(rewards, rewards + B);
  j.seg_off.assign(seg_offsets, seg_offsets + n_seg + 1);
  j.terminal.assign(terminal, terminal + n_seg);
  j.bootstrap.assign(bootstrap, bootstrap + n_seg);
  j.gamma = gamma;
  {
    std::unique_lock<std::mutex> lk(p->mu);
    if (p->error != GA3C_OK) return p->error;
    p->not_full.wait(lk, [&] { return static_cast<int>(p->q.size()) < p->cap || p->closing; });
    if (p->closing) return GA3C_INVALID_ARGUMENT;
    p->q.push_back(std::move(j));
  }
  p->not_empty.notify_one();
  return GA3C_OK;
}

int ga3c_trainer_pool_submit_many(ga3c_trainer_pool* p, int n_batches, const int32_t* batch_off,
                                  const int32_t* seg_base, const int32_t* agents, const int32_t* state_slots,
                                  const int32_t* actions, const double* rewards, const int32_t* seg_offsets,
                                  const uint8_t* terminal, const double* bootstrap, double gamma) {
  if (!p || n_batches < 0 || (n_batches > 0 && (!batch_off || !seg_base || !seg_offsets))) return GA3C_INVALID_ARGUMENT;
  for (int i = 0; i < n_batches; ++i) {
    const int b0 = batch_off[i], s0 = seg_base[i];
    const int st = ga3c_trainer_pool_submit(p, agents + b0, state_slots + b0, batch_off[i + 1] - b0, actions + b0,
                                            rewards + b0, seg_offsets + s0 + i, seg_base[i + 1] - s0, terminal + s0,
                                            bootstrap + s0, gamma);
    if (st != GA3C_OK) return st;
  }
  return GA3C_OK;
}

int ga3c_trainer_pool_wait(ga3c_trainer_pool* p, long long* updates, long long* rejected) {
  if (!p) return GA3C_INVALID_ARGUMENT;
  std::unique_lock<std::mutex> lk(p->mu);
  p->idle.wait(lk, [&] { return p->q.empty() && p->busy == 0; });
  if (updates) *updates = p->updates;
  if (rejected) *rejected = p->rejected;
  return p->error;
}

const char* ga3c_trainer_pool_error(ga3c_trainer_pool* p) {
  // a copy per calling thread: a worker may record the error concurrently
  thread_local std::string msg;
  if (!p) return "";
  std::lock_guard<std::mutex> lk(p->mu);
  msg = p->error_msg;
  return msg.c_str();
}

void ga3c_trainer_pool_destroy(ga3c_trainer_pool* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->closing = true;
  }
  p->not_empty.notify_all();
  p->not_full.notify_all();
  for (auto& t : p->threads) t.join();
  for (auto* c : p->ctxs) ga3c_ctx_destroy(c);
  delete p;
}

}  // extern "C"
