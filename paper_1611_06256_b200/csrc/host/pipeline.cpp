// pipeline.cpp -- the GA3C engine on the B200 C ABI (see ga3c_host.hpp).
//
// Thread structure and stop/shutdown protocol follow the reference engine
// (/root/reference/proj/src/pipeline.cpp:101-612); the math calls go to the
// device: predictors run ga3c_forward_* on a pinned snapshot slot, trainers
// run ga3c_loss_grad_segments_* (device n-step returns + loss/backward) on a
// snapshot and SharedModel::apply (out-of-place RMSProp on the latest slot).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>

#include "ga3c_host.hpp"

namespace ga3c::host {

namespace {

using Clock = std::chrono::steady_clock;
double seconds_between(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

void check(int st, ga3c_model* m, const char* what) {
  if (st == GA3C_OK) return;
  std::string msg = std::string(what) + ": " + ga3c_status_string(st) + " (" + ga3c_model_last_error(m) + ")";
  if (st == GA3C_INVALID_ARGUMENT || st == GA3C_NONFINITE_INPUT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Contexts of retired predictor / trainer threads, kept for the next ones:
// the annealer restarts whole pools when it moves a batch knob, and a new
// context costs its workspace allocation (and its captured graphs).
struct CtxPool {
  std::mutex mu;
  std::vector<std::pair<ga3c_ctx*, int>> free;  // (context, max_batch)
  ~CtxPool() {
    for (auto& e : free) ga3c_ctx_destroy(e.first);
  }
  ga3c_ctx* take(int mb, int* got) {
    std::lock_guard<std::mutex> lk(mu);
    for (std::size_t i = 0; i < free.size(); ++i)
      if (free[i].second >= mb) {
        ga3c_ctx* c = free[i].first;
        *got = free[i].second;
        free.erase(free.begin() + static_cast<std::ptrdiff_t>(i));
        return c;
      }
    return nullptr;
  }
  void give(ga3c_ctx* c, int mb) {
    std::lock_guard<std::mutex> lk(mu);
    free.emplace_back(c, mb);
  }
};

// RAII per-thread device context (stream + workspace), from `pool` when it
// has one large enough and back to it afterwards
struct Ctx {
  ga3c_ctx* c = nullptr;
  int max_batch = 0;
  ga3c_model* m = nullptr;
  CtxPool* pool = nullptr;
  Ctx(ga3c_model* model, int mb, CtxPool* p = nullptr) : m(model), pool(p) {
    if (pool) c = pool->take(mb, &max_batch);
    if (!c) reset(mb);
  }
  ~Ctx() {
    if (!c) return;
    if (pool && ga3c_ctx_sync(c) == GA3C_OK)
      pool->give(c, max_batch);
    else
      ga3c_ctx_destroy(c);
  }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  void reset(int mb) {
    if (c) ga3c_ctx_destroy(c);
    int st = 0;
    c = ga3c_ctx_create(m, mb, &st);
    if (!c) check(st ? st : GA3C_CUDA_ERROR, m, "ga3c_ctx_create");
    max_batch = mb;
  }
  void ensure(int B) {
    if (B > max_batch) reset(std::max(B, 2 * max_batch));
  }
};

// Page-locked host buffer (ga3c_host_alloc): device copies from it are
// asynchronous DMA instead of a staged pageable copy.
struct PinnedBuf {
  std::uint8_t* p = nullptr;
  std::size_t cap = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() { ga3c_host_free(p); }
  std::uint8_t* get(std::size_t bytes) {
    if (bytes > cap) {
      ga3c_host_free(p);
      int st = 0;
      p = static_cast<std::uint8_t*>(ga3c_host_alloc(bytes, &st));
      if (!p) throw std::runtime_error("pinned host allocation failed");
      cap = bytes;
    }
    return p;
  }
};

// Contiguous host batch of observations for one device call.
struct HostBatch {
  bool u8 = false;
  std::vector<std::uint8_t> b8;
  std::vector<float> bf;
  void clear() {
    b8.clear();
    bf.clear();
  }
  void add(const Observation& o) {
    if (u8)
      b8.insert(b8.end(), o.u8.begin(), o.u8.end());
    else
      bf.insert(bf.end(), o.f32.begin(), o.f32.end());
  }
};

// One trainer step on a merged group of agent segments (flush +
// trainer_main math, pipeline.cpp:207-237 / 265-287): device returns, loss
// and gradients on `snap`; the gradient stays in ctx for apply().
void train_on(Ctx& ctx, int slot, const std::vector<ExperienceBatch>& group, const ga3c_hyper& hp,
              HostBatch& hb, std::vector<std::int32_t>& acts, std::vector<double>& rew,
              std::vector<std::int32_t>& off, std::vector<std::uint8_t>& term, std::vector<double>& boot,
              ga3c_frames* frames = nullptr, std::vector<std::int32_t>* fidx = nullptr) {
  hb.clear();
  acts.clear();
  rew.clear();
  off.assign(1, 0);
  term.clear();
  boot.clear();
  if (frames) fidx->clear();
  hb.u8 = !group.front().experiences.front().state.u8.empty();
  for (const auto& b : group) {
    for (const auto& e : b.experiences) {
      if (frames)
        fidx->push_back(e.state_slot);
      else
        hb.add(e.state);
      acts.push_back(e.action);
      rew.push_back(e.reward);
    }
    off.push_back(static_cast<std::int32_t>(acts.size()));
    term.push_back(b.terminal ? 1 : 0);
    boot.push_back(b.terminal ? 0.0 : b.bootstrap);
  }
  const int B = static_cast<int>(acts.size());
  ctx.ensure(B);
  const int n_seg = static_cast<int>(term.size());
  if (frames) {
    // states stay on the device: (agent, slot) per sample
    std::vector<std::int32_t>& ag = *fidx;
    ag.resize(2 * static_cast<std::size_t>(B));
    int k = 0;
    for (const auto& b : group)
      for (std::size_t i = 0; i < b.experiences.size(); ++i) ag[B + k++] = b.agent_id;
    const int st = ga3c_train_frames(ctx.c, slot, frames, ag.data() + B, ag.data(), B, acts.data(), rew.data(),
                                     off.data(), n_seg, term.data(), boot.data(), hp.gamma, 1, nullptr, nullptr);
    check(st, ctx.m, "train_frames");
    return;
  }
  const int st = hb.u8 ? ga3c_loss_grad_segments_u8(ctx.c, slot, hb.b8.data(), B, acts.data(), rew.data(),
                                                    off.data(), n_seg, term.data(), boot.data(), hp.gamma, 1,
                                                    nullptr, nullptr)
                       : ga3c_loss_grad_segments_f32(ctx.c, slot, hb.bf.data(), B, acts.data(), rew.data(),
                                                     off.data(), n_seg, term.data(), boot.data(), hp.gamma, 1,
                                                     nullptr, nullptr);
  check(st, ctx.m, "loss_grad_segments");
}

}  // namespace

// ------------------------------------------------------------ SharedModel
SharedModel::SharedModel(const ga3c_net_spec& spec, const ga3c_hyper& hp, int device, std::uint64_t seed) {
  int st = 0;
  m_ = ga3c_model_create(&spec, &hp, device, &st);
  if (!m_) check(st ? st : GA3C_CUDA_ERROR, nullptr, "ga3c_model_create");
  std::vector<float> th(ga3c_param_count(&spec));
  check(ga3c_init_params(&spec, seed, nullptr, th.data()), m_, "ga3c_init_params");  // nnet.cpp:152-168
  check(ga3c_model_load(m_, th.data(), nullptr, 0), m_, "ga3c_model_load");
}

SharedModel::~SharedModel() { ga3c_model_destroy(m_); }

std::shared_ptr<const SharedModel::Snapshot> SharedModel::snapshot() const {  // pipeline.cpp:22-25
  Snapshot s{};
  check(ga3c_snapshot_acquire(m_, &s.slot, &s.version), m_, "snapshot");
  ga3c_model* m = m_;
  return std::shared_ptr<const Snapshot>(new Snapshot(s), [m](const Snapshot* p) {
    ga3c_snapshot_release(m, p->slot);
    delete p;
  });
}

std::uint64_t SharedModel::version() const { return ga3c_model_version(m_); }

std::optional<std::uint64_t> SharedModel::apply(ga3c_ctx* ctx, const std::function<void(SharedModel&)>& on_applied) {
  std::lock_guard<std::mutex> lk(apply_m_);  // orders on_applied with the publish
  int applied = 0;
  std::uint64_t on = 0;
  const int st = ga3c_apply_rmsprop(ctx, nullptr, &applied, &on);
  if (st == GA3C_NOT_APPLIED) return std::nullopt;  // nnet.cpp:299-301
  check(st, m_, "apply_rmsprop");
  if (on_applied) on_applied(*this);
  return on;
}

std::vector<float> SharedModel::read_theta() const {
  std::vector<float> th(ga3c_model_param_count(m_));
  check(ga3c_model_read(m_, th.data(), nullptr, nullptr), m_, "model_read");
  return th;
}

// -------------------------------------------------------- predictor_loop
void predictor_loop(BoundedChannel<PredictionRequest>& requests,
                    std::vector<std::unique_ptr<ResponseSlot<PredictionResponse>>>& slots,
                    SharedModel& model, ga3c_ctx* ctx, int pred_batch_max, PredictorMetrics& metrics,
                    const std::atomic<bool>& stop, ga3c_frames* frames) {
  std::vector<PredictionRequest> got;
  HostBatch hb;
  std::vector<double> pi, v;
  PinnedBuf newf;
  std::vector<std::int32_t> agents, state_slots;
  std::vector<std::uint8_t> resets;
  while (!stop.load(std::memory_order_relaxed)) {
    auto first = requests.pop(&stop);  // block for the first (pipeline.cpp:72)
    if (!first) break;
    got.clear();
    got.push_back(std::move(*first));
    while (static_cast<int>(got.size()) < pred_batch_max) {  // drain (pipeline.cpp:76-80)
      auto more = requests.try_pop();
      if (!more) break;
      got.push_back(std::move(*more));
    }
    const int B = static_cast<int>(got.size());
    const auto snap = model.snapshot();
    const int A = ga3c_model_n_actions(model.handle());
    pi.resize(static_cast<std::size_t>(B) * A);
    v.resize(B);
    std::uint64_t ver = 0;
    int st;
    if (frames) {
      // newest frames into a pinned batch; the store stacks them on the device
      const std::size_t fb = got.front().state.u8.size();
      std::uint8_t* buf = newf.get(fb * static_cast<std::size_t>(pred_batch_max));
      agents.resize(B);
      resets.resize(B);
      state_slots.resize(B);
      for (int i = 0; i < B; ++i) {
        if (got[i].state.u8.size() != fb) throw std::invalid_argument("predictor: frame size mismatch");
        std::memcpy(buf + static_cast<std::size_t>(i) * fb, got[i].state.u8.data(), fb);
        agents[i] = got[i].agent_id;
        resets[i] = got[i].reset ? 1 : 0;
      }
      st = ga3c_predict_frames64(ctx, snap->slot, frames, buf, agents.data(), resets.data(), B, state_slots.data(),
                                 pi.data(), v.data(), &ver);
    } else {
      hb.u8 = !got.front().state.u8.empty();
      hb.clear();
      for (auto& r : got) hb.add(r.state);
      st = hb.u8 ? ga3c_forward64_u8(ctx, snap->slot, hb.b8.data(), B, pi.data(), v.data(), &ver)
                 : ga3c_forward64_f32(ctx, snap->slot, hb.bf.data(), B, pi.data(), v.data(), &ver);
    }
    check(st, model.handle(), "forward");
    for (int i = 0; i < B; ++i) {
      PredictionResponse resp;
      resp.policy.assign(pi.begin() + static_cast<std::ptrdiff_t>(i) * A,
                         pi.begin() + static_cast<std::ptrdiff_t>(i + 1) * A);
      resp.value = v[i];
      resp.model_version = ver;
      if (frames) resp.state_slot = state_slots[i];
      slots[got[i].agent_id]->put(got[i].ticket, std::move(resp));
    }
    metrics.predictions.fetch_add(B, std::memory_order_relaxed);
    metrics.batches.fetch_add(1, std::memory_order_relaxed);
  }
}

// ---------------------------------------------------------------- validate
void validate(const PipelineOptions& opt) {  // pipeline.cpp:572-603
  check(ga3c_validate_spec(&opt.net), nullptr, "NetworkSpec");
  check(ga3c_validate_hyper(&opt.hyper), nullptr, "Hyperparams");
  validate(opt.env);
  validate(opt.knobs);
  if (!opt.stop.max_updates && !opt.stop.max_seconds && !opt.stop.target_score)
    throw std::invalid_argument("pipeline: no stop condition set");
  if (opt.stop.max_updates && *opt.stop.max_updates < 1)
    throw std::invalid_argument("pipeline: max_updates must be >= 1");
  if (opt.stop.max_seconds && !(*opt.stop.max_seconds > 0.0))
    throw std::invalid_argument("pipeline: max_seconds must be > 0");
  if (!(opt.metrics_interval_s > 0.0)) throw std::invalid_argument("pipeline: metrics interval must be > 0");
  if (opt.anneal) {
    if (!(opt.epoch_s > 0.0)) throw std::invalid_argument("pipeline: epoch length must be > 0");
    if (opt.sync_after_submit) throw std::invalid_argument("pipeline: lockstep mode cannot anneal");
  }
  if (opt.sync_after_submit && (opt.knobs.n_agents != 1 || opt.knobs.n_predictors != 1 ||
                                opt.knobs.n_trainers != 1 || opt.knobs.min_train_batch != 1))
    throw std::invalid_argument(
        "pipeline: lockstep mode requires one agent, one predictor, one trainer and min_train_batch 1");
  auto probe = make_env(opt.env);
  if (opt.device_frames && (!probe->frames() || opt.net.in_c != 4))
    throw std::invalid_argument("pipeline: device frames need an 84x84x4 frame environment");
  const ga3c_net_spec in = probe->input();
  if (in.in_h != opt.net.in_h || in.in_w != opt.net.in_w || in.in_c != opt.net.in_c)
    throw std::invalid_argument("pipeline: net input does not match env observation");
  if (probe->action_count() != opt.net.n_actions)
    throw std::invalid_argument("pipeline: net n_actions does not match env action_count");
}

// ------------------------------------------------------------------ Engine
namespace {

struct Worker {
  std::unique_ptr<std::atomic<bool>> stop;
  std::thread thread;
};

class Engine {
 public:
  explicit Engine(const PipelineOptions& opt)
      : opt_(opt),
        slot_cap_(static_cast<std::size_t>(opt.anneal ? std::max(opt.limits.max_agents, opt.knobs.n_agents)
                                                      : opt.knobs.n_agents)),
        shared_(opt.net, opt.hyper, opt.device, derive_seed(opt.seed, {kSeedModelInit})),
        pred_q_(opt.knobs.pred_queue_cap > 0 ? static_cast<std::size_t>(opt.knobs.pred_queue_cap) : slot_cap_),
        train_q_(static_cast<std::size_t>(opt.knobs.train_queue_cap)),
        budget_(opt.stop.max_updates ? *opt.stop.max_updates : std::numeric_limits<std::int64_t>::max()) {
    for (std::size_t i = 0; i < slot_cap_; ++i) slots_.push_back(std::make_unique<ResponseSlot<PredictionResponse>>());
    if (opt_.device_frames) {
      // Per-agent history of stacked states on the device.  A slot holds a
      // state until the experience made from it is trained or dropped
      // (busy_); an agent whose next slot is still busy hands its open batch
      // to the trainers and waits, so a slot is never rewritten before
      // training read it.  history >= min_train_batch + 2 t_max + 4 lets a
      // stalled agent's experiences always fill the one group in formation.
      const int t = opt_.hyper.t_max;
      const int mtb = opt_.anneal && opt_.anneal_batches ? 1024 : opt_.knobs.min_train_batch;
      hist_ = std::max(256, mtb + 2 * t + 4);
      int st = 0;
      store_ = ga3c_frames_create(shared_.handle(), static_cast<int>(slot_cap_), hist_, &st);
      if (!store_) check(st ? st : GA3C_CUDA_ERROR, shared_.handle(), "ga3c_frames_create");
      busy_ = std::make_unique<std::atomic<std::uint8_t>[]>(slot_cap_ * static_cast<std::size_t>(hist_));
      for (std::size_t i = 0; i < slot_cap_ * static_cast<std::size_t>(hist_); ++i) busy_[i].store(0);
      pushes_.assign(slot_cap_, 0);
    }
    if (opt_.capture_trajectory)
      traj_sink_ = [this](SharedModel& m) {
        std::lock_guard<std::mutex> lk(traj_m_);
        trajectory_.push_back(m.read_theta());
      };
  }

  ~Engine() {
    request_stop();
    join_all();
    ga3c_frames_destroy(store_);
  }

  RunReport run_all() {
    t0_ = Clock::now();
    {
      std::lock_guard<std::mutex> lk(workers_m_);
      for (int i = 0; i < opt_.knobs.n_agents; ++i) add_agent_locked();
      for (int i = 0; i < opt_.knobs.n_predictors; ++i) add_predictor_locked();
      for (int i = 0; i < opt_.knobs.n_trainers; ++i) add_trainer_locked();
    }
    try {
      control_loop();
    } catch (...) {
      report_error(std::current_exception());
    }
    shutdown();
    if (first_error_) std::rethrow_exception(first_error_);
    return make_report();
  }

 private:
  // ---- agents (pipeline.cpp:153-205)
  void agent_main(int id, std::atomic<bool>& stop) {
    try {
      auto env = make_env(opt_.env);
      const bool dev_frames = store_ != nullptr;
      if (dev_frames) env->set_single_frame(true);
      std::mt19937_64 rng(derive_seed(opt_.seed, {kSeedAgentRng, static_cast<std::uint64_t>(id)}));
      std::uint64_t episode = 0;
      Observation obs = env->reset(derive_seed(opt_.seed, {kSeedEnvEpisode, static_cast<std::uint64_t>(id), episode}));
      bool fresh = true;  // the next request starts an episode (device stack = 4 x this frame)
      ExperienceBatch batch;
      batch.agent_id = id;
      double score = 0.0;
      double last_value = 0.0;
      std::int64_t submitted = 0;
      while (!stop.load(std::memory_order_relaxed)) {
        if (dev_frames) {
          // the slot this request's frame is pushed into (only this agent
          // pushes frames for id, pushes_ survives agent restarts)
          std::atomic<std::uint8_t>& next = busy_[slot_of(id, pushes_[id] % hist_)];
          if (next.load(std::memory_order_acquire)) {
            // frame-store backpressure: hand the open batch to the trainers
            // and wait until the experience holding the slot was trained
            if (!batch.experiences.empty() && !flush(batch, false, last_value, stop, submitted)) break;
            while (next.load(std::memory_order_acquire) && !stop.load(std::memory_order_relaxed))
              std::this_thread::yield();
            continue;
          }
        }
        auto& slot = *slots_[id];
        const std::uint64_t ticket = slot.issue_ticket();
        PredictionRequest req{id, ticket, dev_frames ? std::move(obs) : obs, fresh};
        fresh = false;
        if (!pred_q_.push(std::move(req), &stop)) break;
        auto resp = slot.take(ticket, stop);
        if (!resp) break;
        if (dev_frames) ++pushes_[id];
        last_value = resp->value;
        const int A = static_cast<int>(resp->policy.size());
        const int action = opt_.greedy ? argmax_index(resp->policy.data(), A)
                                       : sample_index(resp->policy.data(), A, rng);
        StepResult sr = env->step(action);
        const double reward = opt_.hyper.clip_rewards ? std::clamp(sr.reward, -1.0, 1.0) : sr.reward;
        batch.experiences.push_back(
            Experience{dev_frames ? Observation{} : std::move(obs), action, reward, resp->value, resp->model_version,
                       resp->state_slot});
        if (dev_frames) busy_[slot_of(id, resp->state_slot)].store(1, std::memory_order_release);
        produced_.fetch_add(1, std::memory_order_relaxed);
        score += sr.reward;
        bool ok = true;
        if (sr.terminal) {
          ok = flush(batch, true, 0.0, stop, submitted);
          record_episode(score);
          score = 0.0;
          ++episode;
          obs = env->reset(derive_seed(opt_.seed, {kSeedEnvEpisode, static_cast<std::uint64_t>(id), episode}));
          fresh = true;
        } else {
          obs = std::move(sr.observation);
          if (static_cast<int>(batch.experiences.size()) >= opt_.hyper.t_max)
            ok = flush(batch, false, resp->value, stop, submitted);  // G8: value just played
        }
        if (!ok) break;
      }
      if (!batch.experiences.empty()) {
        dropped_.fetch_add(static_cast<std::int64_t>(batch.experiences.size()));
        release(batch);
      }
    } catch (...) {
      report_error(std::current_exception());
    }
  }

  bool flush(ExperienceBatch& batch, bool terminal, double bootstrap, std::atomic<bool>& stop,
             std::int64_t& submitted) {  // pipeline.cpp:207-237 (returns on the trainer's device)
    batch.terminal = terminal;
    batch.bootstrap = bootstrap;
    ExperienceBatch out;
    out.agent_id = batch.agent_id;
    std::swap(out, batch);
    batch.agent_id = out.agent_id;
    batch.experiences.clear();
    const auto n = static_cast<std::int64_t>(out.experiences.size());
    std::vector<int> held;  // frame-store slots, freed again if the push fails
    if (store_)
      for (const auto& e : out.experiences) held.push_back(e.state_slot);
    if (!train_q_.push(std::move(out), &stop)) {
      dropped_.fetch_add(n);
      for (int sl : held) busy_[slot_of(batch.agent_id, sl)].store(0, std::memory_order_release);
      return false;
    }
    if (opt_.sync_after_submit) {
      ++submitted;
      std::unique_lock<std::mutex> lk(gate_m_);
      gate_cv_.wait(lk, [&] {
        return gate_updates_.load(std::memory_order_relaxed) >= submitted || stop.load(std::memory_order_relaxed);
      });
      if (gate_updates_.load(std::memory_order_relaxed) < submitted) return false;
    }
    return true;
  }

  // ---- trainers (pipeline.cpp:241-306)
  void trainer_main(std::atomic<bool>& stop) {
    try {
      Ctx ctx(shared_.handle(), std::max(64, opt_.knobs.min_train_batch + 4 * opt_.hyper.t_max), &ctx_pool_);
      ga3c_ctx_set_sm_budget(ctx.c, sm_budget(opt_.trainer_sms, 111));
      // trainers are throughput work: one stream-priority level below the
      // predictors, whose forwards the agents wait on (contexts move
      // between roles through ctx_pool_, so both roles set theirs)
      ga3c_ctx_set_priority(ctx.c, 1);
      HostBatch hb;
      std::vector<std::int32_t> acts, off, fidx;
      std::vector<double> rew, boot;
      std::vector<std::uint8_t> term;
      while (!stop.load(std::memory_order_relaxed)) {
        // With the frame store, one trainer at a time forms its group, so at
        // most one group is partly filled and an agent stalled on its
        // history (agent_main) always leaves enough experiences to fill it.
        bool forming = false;
        if (store_) {
          // interruptible: a trainer being retired must not wait behind the
          // one forming a group (that one may wait for agents that wait for
          // predictors the annealer is restarting)
          std::unique_lock<std::mutex> lk(group_m_);
          group_cv_.wait(lk, [&] { return !forming_ || stop.load(std::memory_order_relaxed); });
          if (stop.load(std::memory_order_relaxed)) break;
          forming_ = forming = true;
        }
        auto done_forming = [&] {
          if (!forming) return;
          {
            std::lock_guard<std::mutex> lk(group_m_);
            forming_ = forming = false;
          }
          group_cv_.notify_one();
        };
        auto first = train_q_.pop(&stop);
        if (!first) {
          done_forming();
          break;
        }
        std::vector<ExperienceBatch> group;
        std::int64_t total = static_cast<std::int64_t>(first->experiences.size());
        group.push_back(std::move(*first));
        bool bail = false;
        while (total < opt_.knobs.min_train_batch) {
          auto more = train_q_.pop(&stop);
          if (!more) {
            bail = true;
            break;
          }
          total += static_cast<std::int64_t>(more->experiences.size());
          group.push_back(std::move(*more));
        }
        done_forming();
        if (bail) {
          dropped_.fetch_add(total);
          for (const auto& b : group) release(b);
          break;
        }
        if (budget_.fetch_sub(1, std::memory_order_acq_rel) <= 0) {
          budget_.fetch_add(1, std::memory_order_relaxed);
          dropped_.fetch_add(total);
          for (const auto& b : group) release(b);
          request_stop();
          break;
        }
        const auto snap = shared_.snapshot();
        train_on(ctx, snap->slot, group, opt_.hyper, hb, acts, rew, off, term, boot, store_, &fidx);
        for (const auto& b : group) release(b);  // the device read these states
        const auto applied_on = shared_.apply(ctx.c, traj_sink_);
        if (applied_on) {
          std::uint64_t lag_sum = 0;
          for (const auto& b : group)
            for (const auto& e : b.experiences) lag_sum += *applied_on - e.produced_version;
          bump_gate();
          lag_sum_.fetch_add(lag_sum, std::memory_order_relaxed);
          trained_.fetch_add(total, std::memory_order_relaxed);
          const auto u = updates_.fetch_add(1, std::memory_order_relaxed) + 1;
          if (opt_.stop.max_updates && u >= *opt_.stop.max_updates) request_stop();
        } else {
          budget_.fetch_add(1, std::memory_order_relaxed);
          skipped_.fetch_add(1, std::memory_order_relaxed);
        }
      }
    } catch (...) {
      report_error(std::current_exception());
    }
  }

  // Context SM budget: explicit, or (auto) the device loop's measured split
  // when several trainers share the GPU (trainers 111 of 148 SMs, predictors
  // 64: DESIGN.md section 5), else the whole GPU.
  int sm_budget(int opt, int shared) const {
    if (opt >= 0) return opt;
    return n_t_.load() > 1 ? shared : 0;
  }

  // An experience batch's frame-store states are free again (trained or dropped).
  void release(const ExperienceBatch& b) {
    if (!store_) return;
    for (const auto& e : b.experiences) busy_[slot_of(b.agent_id, e.state_slot)].store(0, std::memory_order_release);
  }
  std::size_t slot_of(int agent, int s) const {
    return static_cast<std::size_t>(agent) * static_cast<std::size_t>(hist_) + static_cast<std::size_t>(s);
  }

  void bump_gate() {
    gate_updates_.fetch_add(1, std::memory_order_relaxed);
    if (opt_.sync_after_submit) {
      std::lock_guard<std::mutex> lk(gate_m_);
      gate_cv_.notify_all();
    }
  }

  // pred_batch_max is the value the thread was started with: the annealer
  // rewrites opt_.knobs before it retires the running predictors, so a
  // predictor reading it live could drain a batch larger than its context
  void predictor_main(std::atomic<bool>& stop, int pred_batch_max) {
    try {
      Ctx ctx(shared_.handle(), pred_batch_max, &ctx_pool_);
      ga3c_ctx_set_sm_budget(ctx.c, sm_budget(opt_.predictor_sms, 64));
      ga3c_ctx_set_priority(ctx.c, 0);
      predictor_loop(pred_q_, slots_, shared_, ctx.c, pred_batch_max, pmetrics_, stop, store_);
    } catch (...) {
      report_error(std::current_exception());
    }
  }

  // ---- worker management (pipeline.cpp:318-407)
  void add_agent_locked() {
    if (stop_requested_.load()) return;
    const int id = next_agent_id_++;
    if (static_cast<std::size_t>(id) >= slot_cap_) throw std::logic_error("pipeline: agent id exceeds slot capacity");
    auto& w = agents_.emplace_back();
    w.stop = std::make_unique<std::atomic<bool>>(false);
    w.thread = std::thread([this, id, s = w.stop.get()] { agent_main(id, *s); });
    n_a_.fetch_add(1);
  }
  void add_predictor_locked() {
    if (stop_requested_.load()) return;
    auto& w = predictors_.emplace_back();
    w.stop = std::make_unique<std::atomic<bool>>(false);
    w.thread = std::thread([this, s = w.stop.get(), pbm = opt_.knobs.pred_batch_max] { predictor_main(*s, pbm); });
    n_p_.fetch_add(1);
  }
  void add_trainer_locked() {
    if (stop_requested_.load()) return;
    auto& w = trainers_.emplace_back();
    w.stop = std::make_unique<std::atomic<bool>>(false);
    w.thread = std::thread([this, s = w.stop.get()] { trainer_main(*s); });
    n_t_.fetch_add(1);
  }
  void remove_last(std::deque<Worker>& pool, std::atomic<std::int64_t>& counter) {
    std::thread t;
    {
      std::lock_guard<std::mutex> lk(workers_m_);
      if (pool.empty()) return;
      pool.back().stop->store(true);
      wake_everything();
      t = std::move(pool.back().thread);
    }
    t.join();
    {
      std::lock_guard<std::mutex> lk(workers_m_);
      pool.pop_back();
      if (&pool == &agents_) --next_agent_id_;
    }
    counter.fetch_sub(1);
  }
  void wake_everything() {
    pred_q_.wake_all();
    train_q_.wake_all();
    {
      std::lock_guard<std::mutex> lk(group_m_);
    }
    group_cv_.notify_all();
    for (auto& s : slots_) s->wake();
    gate_cv_.notify_all();
  }
  void request_stop() {
    std::lock_guard<std::mutex> lk(workers_m_);
    stop_requested_.store(true);
    for (auto* pool : {&agents_, &predictors_, &trainers_})
      for (auto& w : *pool) w.stop->store(true);
    wake_everything();
  }
  void report_error(std::exception_ptr e) {
    {
      std::lock_guard<std::mutex> lk(err_m_);
      if (!first_error_) first_error_ = e;
    }
    request_stop();
  }
  void apply_knobs(const KnobConfig& t) {
    while (n_a_.load() > t.n_agents && !stop_requested_.load()) remove_last(agents_, n_a_);
    while (n_p_.load() > t.n_predictors && !stop_requested_.load()) remove_last(predictors_, n_p_);
    while (n_t_.load() > t.n_trainers && !stop_requested_.load()) remove_last(trainers_, n_t_);
    // batch geometry (only moved with anneal_batches): restart the pools it configures
    if (t.pred_batch_max != live_.pred_batch_max || t.min_train_batch != live_.min_train_batch) {
      live_.pred_batch_max = t.pred_batch_max;
      live_.min_train_batch = t.min_train_batch;
      opt_.knobs.pred_batch_max = t.pred_batch_max;
      opt_.knobs.min_train_batch = t.min_train_batch;
      while (n_p_.load() > 0 && !stop_requested_.load()) remove_last(predictors_, n_p_);
      while (n_t_.load() > 0 && !stop_requested_.load()) remove_last(trainers_, n_t_);
    }
    std::lock_guard<std::mutex> lk(workers_m_);
    while (n_a_.load() < t.n_agents && !stop_requested_.load()) add_agent_locked();
    while (n_p_.load() < t.n_predictors && !stop_requested_.load()) add_predictor_locked();
    while (n_t_.load() < t.n_trainers && !stop_requested_.load()) add_trainer_locked();
  }

  void record_episode(double score) {
    std::lock_guard<std::mutex> lk(scores_m_);
    scores_.push_back(score);
  }
  double rolling_score() {
    std::lock_guard<std::mutex> lk(scores_m_);
    if (scores_.empty()) return 0.0;
    const std::size_t n = std::min<std::size_t>(30, scores_.size());
    double s = 0.0;
    for (std::size_t i = scores_.size() - n; i < scores_.size(); ++i) s += scores_[i];
    return s / static_cast<double>(n);
  }
  std::int64_t n_episodes() {
    std::lock_guard<std::mutex> lk(scores_m_);
    return static_cast<std::int64_t>(scores_.size());
  }

  MetricsFrame frame(double window) {
    MetricsFrame f;
    const auto u = updates_.load(), p = pmetrics_.predictions.load(), b = pmetrics_.batches.load(),
               tr = trained_.load();
    const auto now = Clock::now();
    f.wall_time_s = seconds_between(t0_, now);
    f.tps = (u - last_u_) / window;
    f.pps = (p - last_p_) / window;
    f.samples_per_s = (tr - last_tr_) / window;
    f.pred_batch_mean = b > last_b_ ? static_cast<double>(p - last_p_) / static_cast<double>(b - last_b_) : 0.0;
    f.mean_lag = tr > 0 ? static_cast<double>(lag_sum_.load()) / static_cast<double>(tr) : 0.0;
    f.n_a = static_cast<int>(n_a_.load());
    f.n_p = static_cast<int>(n_p_.load());
    f.n_t = static_cast<int>(n_t_.load());
    f.updates_total = u;
    f.score_mean = rolling_score();
    last_u_ = u;
    last_p_ = p;
    last_b_ = b;
    last_tr_ = tr;
    return f;
  }

  void control_loop() {  // pipeline.cpp:409-479
    using namespace std::chrono_literals;
    live_ = opt_.knobs;
    auto next_frame = t0_ + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(opt_.metrics_interval_s));
    auto last_frame = t0_;
    std::optional<AnnealState> ann;
    std::optional<KnobConfig> cand;
    auto epoch_start = t0_;
    std::int64_t half_updates = -1;
    Clock::time_point half_time;
    if (opt_.anneal)
      ann = make_anneal_state(opt_.knobs, opt_.epoch_s, derive_seed(opt_.seed, {kSeedAnneal}), opt_.limits,
                              opt_.anneal_batches);
    while (!stop_requested_.load()) {
      std::this_thread::sleep_for(2ms);
      {
        std::lock_guard<std::mutex> lk(err_m_);
        if (first_error_) break;
      }
      const auto now = Clock::now();
      if (opt_.stop.max_seconds && seconds_between(t0_, now) >= *opt_.stop.max_seconds) break;
      if (opt_.stop.max_updates && updates_.load() >= *opt_.stop.max_updates) break;
      if (opt_.stop.target_score && n_episodes() >= 30 && rolling_score() >= *opt_.stop.target_score) break;
      if (now >= next_frame) {
        frames_.push_back(frame(seconds_between(last_frame, now)));
        last_frame = now;
        next_frame += std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(opt_.metrics_interval_s));
      }
      if (ann) {
        const double into = seconds_between(epoch_start, now);
        if (half_updates < 0 && into >= opt_.epoch_s / 2.0) {
          half_updates = updates_.load();
          half_time = now;
        } else if (half_updates >= 0 && into >= opt_.epoch_s) {
          const double measured = static_cast<double>(updates_.load() - half_updates) / seconds_between(half_time, now);
          if (!cand) {
            ann->baseline_tps = measured;
            ann->history.push_back(HistoryEntry{ann->current, measured, true});
          } else if (!decide(*ann, *cand, measured)) {
            apply_knobs(ann->current);
          }
          cand = propose(*ann);
          apply_knobs(*cand);
          epoch_start = Clock::now();
          half_updates = -1;
        }
      }
    }
    if (ann) anneal_history_ = ann->history;
    request_stop();
  }

  void join_all() {
    std::vector<std::thread> ts;
    {
      std::lock_guard<std::mutex> lk(workers_m_);
      for (auto* pool : {&agents_, &predictors_, &trainers_})
        for (auto& w : *pool)
          if (w.thread.joinable()) ts.push_back(std::move(w.thread));
    }
    for (auto& t : ts) t.join();
  }

  void shutdown() {
    request_stop();
    join_all();
    frames_.push_back(frame(std::max(1e-9, seconds_between(t0_, Clock::now()))));
    while (auto left = train_q_.try_pop()) left_queued_ += static_cast<std::int64_t>(left->experiences.size());
  }

  RunReport make_report() {
    RunReport r;
    r.total_updates = updates_.load();
    r.skipped_updates = skipped_.load();
    r.total_predictions = pmetrics_.predictions.load();
    {
      std::lock_guard<std::mutex> lk(scores_m_);
      r.total_episodes = static_cast<std::int64_t>(scores_.size());
      r.episode_scores = scores_;
    }
    r.wall_time_s = seconds_between(t0_, Clock::now());
    r.avg_tps = r.total_updates / r.wall_time_s;
    r.avg_pps = r.total_predictions / r.wall_time_s;
    r.experiences_trained = trained_.load();
    r.avg_samples_per_s = r.experiences_trained / r.wall_time_s;
    r.mean_lag = r.experiences_trained > 0 ? static_cast<double>(lag_sum_.load()) / r.experiences_trained : 0.0;
    r.final_knobs = opt_.knobs;
    r.final_knobs.n_agents = static_cast<int>(n_a_.load());
    r.final_knobs.n_predictors = static_cast<int>(n_p_.load());
    r.final_knobs.n_trainers = static_cast<int>(n_t_.load());
    r.final_rolling_score = rolling_score();
    r.frames = frames_;
    r.experiences_produced = produced_.load();
    r.experiences_dropped = dropped_.load();
    r.experiences_left_queued = left_queued_;
    r.anneal_history = anneal_history_;
    {
      std::lock_guard<std::mutex> lk(traj_m_);
      r.theta_trajectory = trajectory_;
    }
    r.final_theta = shared_.read_theta();
    r.final_version = shared_.version();
    return r;
  }

  PipelineOptions opt_;
  std::size_t slot_cap_;
  SharedModel shared_;
  CtxPool ctx_pool_;               // destroyed before shared_'s model (declared after it)
  ga3c_frames* store_ = nullptr;  // device frame store (device_frames)
  int hist_ = 0;
  std::unique_ptr<std::atomic<std::uint8_t>[]> busy_;  // [agent][slot]: holds an untrained experience's state
  std::vector<std::uint64_t> pushes_;                  // frames pushed per agent id
  std::mutex group_m_;                                  // one trainer forms its group at a time:
  std::condition_variable group_cv_;                    // forming_ is set while one does
  bool forming_ = false;
  BoundedChannel<PredictionRequest> pred_q_;
  BoundedChannel<ExperienceBatch> train_q_;
  std::vector<std::unique_ptr<ResponseSlot<PredictionResponse>>> slots_;
  PredictorMetrics pmetrics_;
  KnobConfig live_;

  std::mutex workers_m_;
  std::deque<Worker> agents_, predictors_, trainers_;
  int next_agent_id_ = 0;
  std::atomic<std::int64_t> n_a_{0}, n_p_{0}, n_t_{0};
  std::atomic<bool> stop_requested_{false};
  std::atomic<std::int64_t> gate_updates_{0};
  std::atomic<std::int64_t> budget_;
  std::mutex gate_m_;
  std::condition_variable gate_cv_;

  std::atomic<std::int64_t> updates_{0}, skipped_{0}, produced_{0}, trained_{0}, dropped_{0};
  std::atomic<std::uint64_t> lag_sum_{0};
  std::int64_t last_u_ = 0, last_p_ = 0, last_b_ = 0, last_tr_ = 0;
  std::mutex scores_m_;
  std::vector<double> scores_;

  std::mutex traj_m_;
  std::vector<std::vector<float>> trajectory_;
  std::function<void(SharedModel&)> traj_sink_;

  std::mutex err_m_;
  std::exception_ptr first_error_;
  Clock::time_point t0_;
  std::vector<MetricsFrame> frames_;
  std::vector<HistoryEntry> anneal_history_;
  std::int64_t left_queued_ = 0;
};

}  // namespace

RunReport run(const PipelineOptions& opt) {
  validate(opt);
  Engine e(opt);
  return e.run_all();
}

// reference.cpp:25-157: one thread, zero policy lag, same seeds and the same
// device kernels as the pipeline.
RunReport train_sync(const PipelineOptions& opt) {
  PipelineOptions o = opt;
  o.knobs.n_predictors = 1;
  o.knobs.n_trainers = 1;
  o.knobs.min_train_batch = 1;
  o.sync_after_submit = false;
  o.anneal = false;
  if (!o.stop.max_updates) throw std::invalid_argument("train_sync: max_updates must be set");
  validate(o);
  const auto t0 = Clock::now();
  SharedModel model(o.net, o.hyper, o.device, derive_seed(o.seed, {kSeedModelInit}));
  Ctx ctx(model.handle(), std::max(64, 4 * o.hyper.t_max));
  struct Slot {
    std::unique_ptr<Env> env;
    std::mt19937_64 rng;
    std::uint64_t episode = 0;
    Observation obs;
    double score = 0.0;
  };
  const int n_agents = o.knobs.n_agents;
  std::vector<Slot> agents(n_agents);
  for (int i = 0; i < n_agents; ++i) {
    agents[i].env = make_env(o.env);
    agents[i].rng.seed(derive_seed(o.seed, {kSeedAgentRng, static_cast<std::uint64_t>(i)}));
    agents[i].obs = agents[i].env->reset(derive_seed(o.seed, {kSeedEnvEpisode, static_cast<std::uint64_t>(i), 0}));
  }
  RunReport rep;
  HostBatch hb, one;
  std::vector<std::int32_t> acts, off;
  std::vector<double> rew, boot;
  std::vector<std::uint8_t> term;
  const int A = o.net.n_actions;
  std::vector<double> pi(A);
  double v = 0.0;
  int turn = 0;
  while (rep.total_updates < *o.stop.max_updates) {
    Slot& a = agents[turn];
    const int agent_id = turn;
    turn = (turn + 1) % n_agents;
    ExperienceBatch batch;
    batch.agent_id = agent_id;
    while (true) {
      const auto snap = model.snapshot();
      std::uint64_t ver = 0;
      const bool u8 = !a.obs.u8.empty();
      const int st = u8 ? ga3c_forward64_u8(ctx.c, snap->slot, a.obs.u8.data(), 1, pi.data(), &v, &ver)
                        : ga3c_forward64_f32(ctx.c, snap->slot, a.obs.f32.data(), 1, pi.data(), &v, &ver);
      check(st, model.handle(), "forward");
      rep.total_predictions += 1;
      const int action = o.greedy ? argmax_index(pi.data(), A) : sample_index(pi.data(), A, a.rng);
      StepResult sr = a.env->step(action);
      const double reward = o.hyper.clip_rewards ? std::clamp(sr.reward, -1.0, 1.0) : sr.reward;
      batch.experiences.push_back(Experience{std::move(a.obs), action, reward, v, ver});
      rep.experiences_produced += 1;
      a.score += sr.reward;
      if (sr.terminal) {
        batch.terminal = true;
        rep.episode_scores.push_back(a.score);
        a.score = 0.0;
        ++a.episode;
        a.obs = a.env->reset(derive_seed(o.seed, {kSeedEnvEpisode, static_cast<std::uint64_t>(agent_id), a.episode}));
        break;
      }
      a.obs = std::move(sr.observation);
      if (static_cast<int>(batch.experiences.size()) >= o.hyper.t_max) {
        batch.bootstrap = v;  // the value just played seeds the tail (G8)
        break;
      }
    }
    const auto snap = model.snapshot();
    std::vector<ExperienceBatch> group;
    group.push_back(std::move(batch));
    train_on(ctx, snap->slot, group, o.hyper, hb, acts, rew, off, term, boot);
    if (model.apply(ctx.c)) {
      rep.total_updates += 1;
      rep.experiences_trained += static_cast<std::int64_t>(acts.size());
      if (o.capture_trajectory) rep.theta_trajectory.push_back(model.read_theta());
    } else {
      rep.skipped_updates += 1;
    }
  }
  rep.total_episodes = static_cast<std::int64_t>(rep.episode_scores.size());
  rep.wall_time_s = seconds_between(t0, Clock::now());
  rep.avg_tps = rep.total_updates / rep.wall_time_s;
  rep.avg_pps = rep.total_predictions / rep.wall_time_s;
  rep.avg_samples_per_s = rep.experiences_trained / rep.wall_time_s;
  rep.final_knobs = o.knobs;
  if (!rep.episode_scores.empty()) {
    const std::size_t n = std::min<std::size_t>(30, rep.episode_scores.size());
    double s = 0.0;
    for (std::size_t i = rep.episode_scores.size() - n; i < rep.episode_scores.size(); ++i) s += rep.episode_scores[i];
    rep.final_rolling_score = s / static_cast<double>(n);
  }
  rep.final_theta = model.read_theta();
  rep.final_version = model.version();
  return rep;
}

}  // namespace ga3c::host
