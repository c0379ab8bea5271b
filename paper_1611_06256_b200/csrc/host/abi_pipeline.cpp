// abi_pipeline.cpp -- C ABI of the host engine (include/ga3c.h, "pipeline"):
// the flat-struct face of ga3c::host::run / train_sync that a binding (the
// reference's qac.run / qac.train_sync, qac_module.cpp:255-294) calls with the
// GIL released.
#include <cstring>
#include <exception>
#include <string>

#include "ga3c.h"
#include "ga3c_host.hpp"

using namespace ga3c::host;

namespace {

PipelineOptions to_options(const ga3c_pipeline_opts* o) {
  PipelineOptions p;
  p.net = o->net;
  p.hyper = o->hyper;
  p.env.kind = static_cast<EnvKind>(o->env_kind);
  p.env.n_contexts = o->n_contexts;
  p.env.n_actions = o->env_actions;
  p.env.grid_size = o->grid_size;
  p.env.step_delay_us = o->step_delay_us;
  p.env.episode_len = o->episode_len;
  p.env.action_repeat = o->action_repeat;
  p.knobs.n_agents = o->n_agents;
  p.knobs.n_predictors = o->n_predictors;
  p.knobs.n_trainers = o->n_trainers;
  p.knobs.pred_batch_max = o->pred_batch_max;
  p.knobs.min_train_batch = o->min_train_batch;
  p.knobs.train_queue_cap = o->train_queue_cap;
  p.knobs.pred_queue_cap = o->pred_queue_cap;
  if (o->max_updates > 0) p.stop.max_updates = o->max_updates;
  if (o->max_seconds > 0.0) p.stop.max_seconds = o->max_seconds;
  if (o->has_target_score) p.stop.target_score = o->target_score;
  p.seed = o->seed;
  p.anneal = o->anneal != 0;
  p.anneal_batches = o->anneal_batches != 0;
  p.epoch_s = o->epoch_s;
  p.limits.max_agents = o->max_agents;
  p.limits.max_predictors = o->max_predictors;
  p.limits.max_trainers = o->max_trainers;
  p.metrics_interval_s = o->metrics_interval_s;
  p.greedy = o->greedy != 0;
  p.sync_after_submit = o->sync_after_submit != 0;
  p.capture_trajectory = o->capture_trajectory != 0;
  p.device = o->device;
  p.device_frames = o->device_frames != 0;
  p.trainer_sms = o->trainer_sms;
  p.predictor_sms = o->predictor_sms;
  return p;
}

}  // namespace

extern "C" {

void ga3c_default_pipeline_opts(ga3c_pipeline_opts* o) {
  std::memset(o, 0, sizeof(*o));
  ga3c_default_hyper(&o->hyper);
  o->env_kind = 0;
  o->n_contexts = 4;
  o->env_actions = 4;
  o->grid_size = 5;
  o->step_delay_us = 500;
  o->episode_len = 64;
  o->action_repeat = 1;
  const KnobConfig k;
  o->n_agents = k.n_agents;
  o->n_predictors = k.n_predictors;
  o->n_trainers = k.n_trainers;
  o->pred_batch_max = k.pred_batch_max;
  o->min_train_batch = k.min_train_batch;
  o->train_queue_cap = k.train_queue_cap;
  o->pred_queue_cap = k.pred_queue_cap;
  o->seed = 1;
  o->epoch_s = 60.0;
  const Limits l;
  o->max_agents = l.max_agents;
  o->max_predictors = l.max_predictors;
  o->max_trainers = l.max_trainers;
  o->metrics_interval_s = 1.0;
  o->trainer_sms = -1;
  o->predictor_sms = -1;
}

int ga3c_pipeline_run(const ga3c_pipeline_opts* o, int sync_trainer, ga3c_run_report* r, float* final_theta,
                      float* trajectory, int traj_cap, double* episode_scores, int scores_cap,
                      ga3c_anneal_entry* anneal, int anneal_cap, char* err, int err_len) {
  auto set_err = [&](const char* msg) {
    if (err && err_len > 0) {
      std::strncpy(err, msg, static_cast<std::size_t>(err_len) - 1);
      err[err_len - 1] = '\0';
    }
  };
  if (!o || !r) return GA3C_INVALID_ARGUMENT;
  try {
    const PipelineOptions p = to_options(o);
    const RunReport rep = sync_trainer ? train_sync(p) : run(p);
    std::memset(r, 0, sizeof(*r));
    r->total_updates = rep.total_updates;
    r->skipped_updates = rep.skipped_updates;
    r->total_predictions = rep.total_predictions;
    r->total_episodes = rep.total_episodes;
    r->wall_time_s = rep.wall_time_s;
    r->avg_tps = rep.avg_tps;
    r->avg_pps = rep.avg_pps;
    r->avg_samples_per_s = rep.avg_samples_per_s;
    r->mean_lag = rep.mean_lag;
    r->final_rolling_score = rep.final_rolling_score;
    r->experiences_produced = rep.experiences_produced;
    r->experiences_trained = rep.experiences_trained;
    r->experiences_dropped = rep.experiences_dropped;
    r->experiences_left_queued = rep.experiences_left_queued;
    r->final_n_agents = rep.final_knobs.n_agents;
    r->final_n_predictors = rep.final_knobs.n_predictors;
    r->final_n_trainers = rep.final_knobs.n_trainers;
    r->final_pred_batch_max = rep.final_knobs.pred_batch_max;
    r->final_min_train_batch = rep.final_knobs.min_train_batch;
    r->final_version = rep.final_version;
    r->n_trajectory = static_cast<int>(rep.theta_trajectory.size());
    r->n_anneal = static_cast<int>(rep.anneal_history.size());
    r->n_frames = static_cast<int>(rep.frames.size());
    if (!rep.frames.empty()) {
      r->last_frame_tps = rep.frames.back().tps;
      r->last_frame_pps = rep.frames.back().pps;
      r->last_frame_pred_batch_mean = rep.frames.back().pred_batch_mean;
    }
    const std::size_t P = rep.final_theta.size();
    if (final_theta) std::memcpy(final_theta, rep.final_theta.data(), P * sizeof(float));
    if (trajectory)
      for (int i = 0; i < traj_cap && i < r->n_trajectory; ++i)
        std::memcpy(trajectory + static_cast<std::size_t>(i) * P, rep.theta_trajectory[i].data(), P * sizeof(float));
    if (episode_scores)
      for (int i = 0; i < scores_cap && i < static_cast<int>(rep.episode_scores.size()); ++i)
        episode_scores[i] = rep.episode_scores[i];
    if (anneal)
      for (int i = 0; i < anneal_cap && i < r->n_anneal; ++i) {
        const auto& h = rep.anneal_history[i];
        anneal[i].n_agents = h.knobs.n_agents;
        anneal[i].n_predictors = h.knobs.n_predictors;
        anneal[i].n_trainers = h.knobs.n_trainers;
        anneal[i].pred_batch_max = h.knobs.pred_batch_max;
        anneal[i].min_train_batch = h.knobs.min_train_batch;
        anneal[i].measured_tps = h.measured_tps;
        anneal[i].accepted = h.accepted ? 1 : 0;
      }
    return GA3C_OK;
  } catch (const std::invalid_argument& e) {
    set_err(e.what());
    return GA3C_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    set_err(e.what());
    return GA3C_CUDA_ERROR;
  }
}

}  // extern "C"
