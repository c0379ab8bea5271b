// ga3c_host.hpp -- C++ host side of the B200 GA3C hot path.
//
// Mirrors the reference engine (/root/reference/proj/include/qac/pipeline.hpp,
// envs.hpp, annealer.hpp, knobs.hpp, util.hpp) on top of the C ABI
// (include/ga3c.h): agent threads step CPU environments and push
// PredictionRequests; predictor threads drain the PredictionQueue into one
// batched device forward on an immutable parameter snapshot
// (predictor_loop, pipeline.cpp:65-93); trainer threads coalesce the
// TrainingQueue to min_train_batch and run returns + loss/backward on a
// snapshot, then apply RMSProp to the LATEST parameters through the device
// SharedModel (pipeline.cpp:241-306, 37-63); a control thread owns stop
// conditions, metric frames and the annealer (pipeline.cpp:409-479).
// train_sync is the zero-lag single-thread trainer (reference.cpp:25-157)
// running the same device kernels, so a lockstep pipeline reproduces it bit
// for bit (the kernels are deterministic).
#pragma once

#include <atomic>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "channel.hpp"
#include "ga3c.h"

namespace ga3c::host {

// ------------------------------------------------------------- util.hpp
std::uint64_t mix64(std::uint64_t x);
std::uint64_t derive_seed(std::uint64_t base, std::initializer_list<std::uint64_t> salts);
inline constexpr std::uint64_t kSeedModelInit = 0x6d6f64656cULL;  // util.hpp:34
inline constexpr std::uint64_t kSeedAgentRng = 0x6167656e74ULL;   // util.hpp:35
inline constexpr std::uint64_t kSeedEnvEpisode = 0x656e76ULL;     // util.hpp:36
inline constexpr std::uint64_t kSeedAnneal = 0x616e6e65616cULL;   // pipeline.cpp:13
double next_uniform(std::mt19937_64& rng);                         // util.hpp:41-43
int sample_index(const double* probs, int n, std::mt19937_64& rng);  // util.hpp:46-54 (fp64 CDF)
int argmax_index(const double* values, int n);                     // util.hpp:57-63
void busy_wait_us(std::int64_t us);

// ------------------------------------------------------------- envs.hpp
enum class EnvKind { ContextualBandit = 0, Catch = 1, DelayLab = 2, FrameCatch = 3, Frames = 4 };

struct EnvSpec {
  EnvKind kind = EnvKind::ContextualBandit;
  int n_contexts = 4;
  int n_actions = 4;
  int grid_size = 5;
  std::int64_t step_delay_us = 500;
  int episode_len = 64;
  int action_repeat = 1;
};

struct Observation {  // exactly one of the two is used, by env kind
  std::vector<float> f32;
  std::vector<std::uint8_t> u8;
};

struct StepResult {
  Observation observation;
  double reward = 0.0;
  bool terminal = false;
};

class Env {
 public:
  virtual ~Env() = default;
  virtual Observation reset(std::uint64_t seed) = 0;
  virtual StepResult step(int action) = 0;
  virtual int action_count() const = 0;
  virtual bool frames() const = 0;       // u8 84x84x4 observations
  virtual ga3c_net_spec input() const = 0;  // in_h/in_w/in_c of the observation
  // Device frame store mode (frame envs only): observations carry only the
  // NEWEST frame (in_h x in_w bytes); the 4-frame stack is built on the
  // device (ga3c_predict_frames), where it equals the stack frames() mode
  // returns (reset = the first frame four times).
  virtual void set_single_frame(bool on) {
    if (on) throw std::invalid_argument("env: no single-frame observations");
  }
};

void validate(const EnvSpec& spec);
std::unique_ptr<Env> make_env(const EnvSpec& spec);

// ------------------------------------------------------------ knobs.hpp
struct KnobConfig {
  int n_agents = 1;
  int n_predictors = 2;
  int n_trainers = 2;
  int pred_batch_max = 32;
  int min_train_batch = 1;
  int train_queue_cap = 32;
  int pred_queue_cap = 0;  // 0 = one slot per agent
  bool operator==(const KnobConfig&) const = default;
};
void validate(const KnobConfig& k);

// --------------------------------------------------------- annealer.hpp
struct Limits {
  int max_agents = 64;
  int max_predictors = 16;
  int max_trainers = 16;
};
struct HistoryEntry {
  KnobConfig knobs;
  double measured_tps = 0.0;
  bool accepted = false;
};
struct AnnealState {
  KnobConfig current;
  double baseline_tps = 0.0;
  double epoch_length_s = 60.0;
  double baseline_decay = 0.01;
  Limits limits;
  bool tune_batches = false;  // extension: also move pred_batch_max / min_train_batch
  std::mt19937_64 rng;
  std::vector<HistoryEntry> history;
};
AnnealState make_anneal_state(const KnobConfig& initial, double epoch_length_s, std::uint64_t seed,
                              const Limits& limits, bool tune_batches = false);
KnobConfig propose(AnnealState& s);                                        // annealer.cpp:28-53
bool decide(AnnealState& s, const KnobConfig& candidate, double measured_tps);  // annealer.cpp:55-66

// ------------------------------------------------------------ pipeline
struct PredictionRequest {
  int agent_id = 0;
  std::uint64_t ticket = 0;
  Observation state;  // device frames: the newest frame only
  bool reset = false;  // device frames: first frame of an episode
};

struct PredictionResponse {
  std::vector<double> policy;  // the device's fp64 softmax (ga3c_forward64_*)
  double value = 0.0;
  std::uint64_t model_version = 0;
  int state_slot = -1;  // device frames: where the stacked state is kept
};

struct Experience {  // returns.hpp:13-19
  Observation state;    // empty with device frames
  int action = 0;
  double reward = 0.0;
  double value_at_play = 0.0;
  std::uint64_t produced_version = 0;
  int state_slot = -1;  // device frames: the state's slot in the agent's ring
};

struct ExperienceBatch {  // returns.hpp:21-26 (returns computed on the trainer's device)
  std::vector<Experience> experiences;
  bool terminal = false;
  double bootstrap = 0.0;
  int agent_id = 0;
};

struct StopCondition {
  std::optional<std::int64_t> max_updates;
  std::optional<double> max_seconds;
  std::optional<double> target_score;
};

struct MetricsFrame {
  double wall_time_s = 0.0, tps = 0.0, pps = 0.0, samples_per_s = 0.0, mean_lag = 0.0;
  double pred_batch_mean = 0.0;
  int n_a = 0, n_p = 0, n_t = 0;
  std::int64_t updates_total = 0;
  double score_mean = 0.0;
};

struct RunReport {
  std::int64_t total_updates = 0, skipped_updates = 0, total_predictions = 0, total_episodes = 0;
  double wall_time_s = 0.0, avg_tps = 0.0, avg_pps = 0.0, avg_samples_per_s = 0.0, mean_lag = 0.0;
  KnobConfig final_knobs;
  double final_rolling_score = 0.0;
  std::vector<double> episode_scores;
  std::vector<MetricsFrame> frames;
  std::int64_t experiences_produced = 0, experiences_trained = 0, experiences_dropped = 0,
               experiences_left_queued = 0;
  std::vector<HistoryEntry> anneal_history;
  std::vector<std::vector<float>> theta_trajectory;
  std::vector<float> final_theta;
  std::uint64_t final_version = 0;
};

struct PipelineOptions {  // pipeline.hpp:67-85
  ga3c_net_spec net{};
  ga3c_hyper hyper{};
  EnvSpec env;
  KnobConfig knobs;
  StopCondition stop;
  std::uint64_t seed = 1;
  bool anneal = false;
  bool anneal_batches = false;
  double epoch_s = 60.0;
  Limits limits;
  double metrics_interval_s = 1.0;
  bool greedy = false;
  bool sync_after_submit = false;
  bool capture_trajectory = false;
  int device = 0;
  // Device frame store (ga3c_frames_*, frame envs): agents send only their
  // newest 84x84 frame, the stacks live on the GPU, and the TrainingQueue
  // carries frame-store slots instead of 28 KB states.
  bool device_frames = false;
  // SM budgets of trainer / predictor contexts: -1 automatic, 0 all, n SMs
  int trainer_sms = -1;
  int predictor_sms = -1;
};

// Device-resident SharedModel (pipeline.hpp:92-111): immutable snapshots are
// pinned parameter slots of the ga3c_model ring; apply() writes the RMSProp
// step out of place onto the latest slot and publishes it.
class SharedModel {
 public:
  SharedModel(const ga3c_net_spec& spec, const ga3c_hyper& hp, int device, std::uint64_t init_seed);
  ~SharedModel();
  SharedModel(const SharedModel&) = delete;
  SharedModel& operator=(const SharedModel&) = delete;

  struct Snapshot {
    int slot;
    std::uint64_t version;
  };
  std::shared_ptr<const Snapshot> snapshot() const;
  std::uint64_t version() const;
  // RMSProp on the latest parameters from the gradient held in `ctx`;
  // returns the version it applied on top of, nothing when rejected.
  std::optional<std::uint64_t> apply(ga3c_ctx* ctx, const std::function<void(SharedModel&)>& on_applied = {});
  std::vector<float> read_theta() const;
  ga3c_model* handle() const { return m_; }

 private:
  ga3c_model* m_ = nullptr;
  std::mutex apply_m_;
};

// predictor_loop (pipeline.hpp:117-120 / pipeline.cpp:65-93): block for the
// first request, drain up to pred_batch_max, one device forward on one
// snapshot, route every response by ticket.
struct PredictorMetrics {
  std::atomic<std::int64_t> predictions{0};
  std::atomic<std::int64_t> batches{0};
};
// frames (nullable): requests carry newest frames, pushed into the device
// frame store by the batched forward (ga3c_predict_frames64).
void predictor_loop(BoundedChannel<PredictionRequest>& requests,
                    std::vector<std::unique_ptr<ResponseSlot<PredictionResponse>>>& slots,
                    SharedModel& model, ga3c_ctx* ctx, int pred_batch_max, PredictorMetrics& metrics,
                    const std::atomic<bool>& stop, ga3c_frames* frames = nullptr);

void validate(const PipelineOptions& opt);
RunReport run(const PipelineOptions& opt);          // pipeline.cpp:607-611
RunReport train_sync(const PipelineOptions& opt);   // reference.cpp:25-157 (n_agents round robin)

}  // namespace ga3c::host
