/*
 * ga3c.h -- C ABI of the B200-native GA3C hot path (libga3c_b200.so).
 *
 * This is the drop-in boundary for the reference `qac` library's math layer
 * (/root/reference/proj/include/qac/nnet.hpp:66-104, returns.hpp:31-32) and
 * for the device side of its SharedModel / predictor / trainer
 * (pipeline.hpp:92-120).  Every entry point names the reference interface it
 * replaces.  Conventions:
 *   - plain C types only: pointers + sizes, no torch or STL types;
 *   - int status codes, never exceptions across the ABI.  The C++ adapter
 *     (paper_1611_06256_b200/csrc/host/qac_b200.hpp) rethrows
 *     GA3C_INVALID_ARGUMENT as std::invalid_argument, like the reference;
 *   - caller-owned host buffers, library-owned device buffers;
 *   - one ga3c_model per device (parameters + RMSProp state, versioned
 *     snapshots); one ga3c_ctx per predictor/trainer thread (its own CUDA
 *     stream + workspace).  Calls on distinct contexts may run concurrently;
 *     apply is serialized inside the model (pipeline.cpp:40).
 *   - arithmetic is fp32 on the device (reference: fp64); parity tolerances
 *     are stated in DESIGN.md and tests/.  Returns are fp64, bitwise.
 * There is no CPU fallback: without a usable sm_100 device every compute
 * call returns GA3C_CUDA_ERROR.
 */
#ifndef GA3C_H
#define GA3C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GA3C_MAX_CONV 4
#define GA3C_MAX_HIDDEN 4

/* Status codes. */
#define GA3C_OK 0
#define GA3C_INVALID_ARGUMENT 1 /* reference: std::invalid_argument */
#define GA3C_NONFINITE_INPUT 2  /* reference: std::invalid_argument (non-finite state/return) */
#define GA3C_CUDA_ERROR 3
#define GA3C_NCCL_ERROR 4
#define GA3C_NOT_APPLIED 5      /* rmsprop rejected a non-finite gradient (nnet.cpp:299-301) */
#define GA3C_OUT_OF_MEMORY 6

/* Network spec.  Extends NetworkSpec (nnet.hpp:14-18) with VALID NHWC conv
 * layers.  The reference's {input_dim, hidden_dims, n_actions}
 * is in_h = in_w = 1, in_c = input_dim, n_conv = 0; its flat parameter layout
 * (nnet.cpp:29-45) is reproduced exactly, conv layers first as
 * W[Cout][k][k][Cin] (OHWI) then b[Cout]; FC layers consume the NHWC flatten. */
typedef struct ga3c_net_spec {
  int in_h, in_w, in_c;
  int n_conv;
  int conv_out[GA3C_MAX_CONV];
  int conv_k[GA3C_MAX_CONV];
  int conv_stride[GA3C_MAX_CONV];
  int n_hidden;
  int hidden[GA3C_MAX_HIDDEN];
  int n_actions;
} ga3c_net_spec;

/* Hyperparams (nnet.hpp:20-31), same field order and defaults. */
typedef struct ga3c_hyper {
  double gamma;             /* 0.99 */
  int t_max;                /* 5 */
  double beta;              /* 0.01 entropy bonus */
  double eps_log;           /* 1e-6 */
  double eta;               /* 3e-4 */
  double alpha;             /* 0.99 rmsprop decay */
  double eps_rms;           /* 1e-8 */
  double value_loss_weight; /* 0.5 */
  double grad_clip_norm;    /* 0 = off */
  int clip_rewards;         /* 0 */
} ga3c_hyper;

typedef struct ga3c_model ga3c_model;
typedef struct ga3c_ctx ga3c_ctx;

const char* ga3c_status_string(int status);
void ga3c_default_hyper(ga3c_hyper* hp);

/* ---------------------------------------------------- spec and layout */
/* nnet::validate(NetworkSpec) nnet.cpp:123-130 / validate(Hyperparams) :131-145 */
int ga3c_validate_spec(const ga3c_net_spec* spec);
int ga3c_validate_hyper(const ga3c_hyper* hp);
/* nnet::param_count nnet.hpp:71 (0 if the spec is invalid) */
size_t ga3c_param_count(const ga3c_net_spec* spec);
size_t ga3c_input_dim(const ga3c_net_spec* spec);
/* nnet::init_model nnet.hpp:75 / nnet.cpp:152-168 (host, mt19937_64).
 * theta64 (nullable) receives the fp64 draws, theta32 (nullable) their fp32
 * rounding -- the values the device computes with. */
int ga3c_init_params(const ga3c_net_spec* spec, uint64_t seed, double* theta64, float* theta32);

/* ------------------------------------------- SharedModel (device side) */
/* SharedModel ctor pipeline.hpp:94: params + rms accumulator live on `device`. */
ga3c_model* ga3c_model_create(const ga3c_net_spec* spec, const ga3c_hyper* hp, int device,
                              int* status);
void ga3c_model_destroy(ga3c_model* m);
/* Install theta (fp32, P values), g (nullable = zeros, init_rms nnet.cpp:170)
 * and version as a new snapshot. */
int ga3c_model_load(ga3c_model* m, const float* theta, const float* g, uint64_t version);
/* Copy parameter slot `slot` (theta and/or g, nullable) to the host after
 * every write to it in flight on any stream (device synchronise). */
int ga3c_model_read_slot(ga3c_model* m, int slot, float* theta, float* g);
/* Copy the latest snapshot out (ModelState/RmsState nnet.hpp:35-44). */
int ga3c_model_read(ga3c_model* m, float* theta, float* g, uint64_t* version);
/* SharedModel::version pipeline.hpp:98 */
uint64_t ga3c_model_version(ga3c_model* m);
size_t ga3c_model_param_count(ga3c_model* m);
int ga3c_model_n_actions(ga3c_model* m);
/* SharedModel::snapshot pipeline.hpp:96: pin the latest immutable parameter
 * slot; it cannot be recycled until released. */
int ga3c_snapshot_acquire(ga3c_model* m, int* slot, uint64_t* version);
int ga3c_snapshot_release(ga3c_model* m, int slot);
const char* ga3c_model_last_error(ga3c_model* m);

/* ------------------------------------------------ per-thread contexts */
ga3c_ctx* ga3c_ctx_create(ga3c_model* m, int max_batch, int* status);
void ga3c_ctx_destroy(ga3c_ctx* c);
void* ga3c_ctx_stream(ga3c_ctx* c); /* cudaStream_t */
int ga3c_ctx_sync(ga3c_ctx* c);
/* Number of kernels this context has launched (evidence counter). */
uint64_t ga3c_ctx_launches(ga3c_ctx* c);

/* ------------------------------------------------------------ forward */
/* nnet::forward nnet.hpp:81 / nnet.cpp:174-191 on snapshot `slot` (-1 =
 * latest, pinned for the call).  Host buffers, blocking.  States are NHWC;
 * u8 frames mean x = k/256 (exact in fp32).  pi: B x n_actions, v: B.
 * version_used (nullable) receives the snapshot version (PredictionResponse
 * model_version, pipeline.hpp:32). */
int ga3c_forward_u8(ga3c_ctx* c, int slot, const uint8_t* frames, int B, float* pi, float* v,
                    uint64_t* version_used);
int ga3c_forward_f32(ga3c_ctx* c, int slot, const float* states, int B, float* pi, float* v,
                     uint64_t* version_used);
/* The same with the policy as the device's fp64 softmax (the reference's
 * ForwardResult.policies type, nnet.hpp:55-58): pi rows sum to 1 within fp64
 * rounding, and qac::sample_index (util.hpp:46-54) on them draws exactly the
 * action ga3c_sample_actions_dev draws on the device.  v = V widened to fp64. */
int ga3c_forward64_u8(ga3c_ctx* c, int slot, const uint8_t* frames, int B, double* pi, double* v,
                      uint64_t* version_used);
int ga3c_forward64_f32(ga3c_ctx* c, int slot, const float* states, int B, double* pi, double* v,
                       uint64_t* version_used);
/* Device-resident variant: all pointers are device memory; asynchronous on
 * the context stream; `slot` must be pinned by the caller.  state_stride =
 * elements between consecutive states (0 = dense), so a batch can be read
 * straight out of a per-agent frame ring.  d_pi / d_v (nullable) receive
 * copies; the sampler can also read the context's own last output. */
int ga3c_forward_dev(ga3c_ctx* c, int slot, const void* d_states, int states_are_u8,
                     long long state_stride, int B, float* d_pi, float* d_v);

/* --------------------------------------------------- loss + gradients */
/* nnet::loss_and_gradients nnet.hpp:94 / nnet.cpp:201-291 on snapshot `slot`.
 * Summed (not averaged) gradient over the batch; the result stays in the
 * context's gradient buffer and is copied to dtheta (nullable).
 * scalars (nullable) = {policy_loss, value_loss, entropy}.  apply_clip = 0
 * defers the optional global-norm clip (nnet.cpp:281-289) so a data-parallel
 * caller can clip after the allreduce (ga3c_clip_grad). */
int ga3c_loss_grad_u8(ga3c_ctx* c, int slot, const uint8_t* frames, const int32_t* actions,
                      const double* returns, int B, int apply_clip, float* dtheta,
                      double* scalars);
int ga3c_loss_grad_f32(ga3c_ctx* c, int slot, const float* states, const int32_t* actions,
                       const double* returns, int B, int apply_clip, float* dtheta,
                       double* scalars);
/* Device-resident variant (async); all pointers are device memory.  Actions
 * are not validated on the host: a sample whose action is outside
 * [0, n_actions) makes the gradient non-finite, so the following apply
 * rejects the step (the reference throws, nnet.cpp:227-228). */
int ga3c_loss_grad_dev(ga3c_ctx* c, int slot, const void* d_states, int states_are_u8,
                       long long state_stride, const int32_t* d_actions, const double* d_returns,
                       int B, int apply_clip);
/* Trainer step with on-device n-step returns: the merged batch of n_seg
 * agent segments (segment s = rows seg_offsets[s] .. seg_offsets[s+1]) is
 * uploaded with its rewards, terminal flags and bootstrap values;
 * returns::compute_returns (returns.cpp:8-26) runs per segment on the device
 * and feeds loss_and_gradients (nnet.cpp:201-291) directly.  Equivalent to
 * the reference's flush() + trainer_main() pair (pipeline.cpp:207-306).
 * returns_out (nullable) receives the fp64 returns. */
int ga3c_loss_grad_segments_u8(ga3c_ctx* c, int slot, const uint8_t* frames, int B,
                               const int32_t* actions, const double* rewards,
                               const int32_t* seg_offsets, int n_seg, const uint8_t* terminal,
                               const double* bootstrap, double gamma, int apply_clip,
                               double* scalars, double* returns_out);
int ga3c_loss_grad_segments_f32(ga3c_ctx* c, int slot, const float* states, int B,
                                const int32_t* actions, const double* rewards,
                                const int32_t* seg_offsets, int n_seg, const uint8_t* terminal,
                                const double* bootstrap, double gamma, int apply_clip,
                                double* scalars, double* returns_out);
/* The context's device gradient buffer (P floats) -- e.g. for an NCCL
 * allreduce(sum) across data-parallel replicas. */
float* ga3c_ctx_grad(ga3c_ctx* c);
/* The context's fp64 copy of the last forward's values V (device, B
 * doubles): the bootstrap input of ga3c_compute_returns_dev (the reference
 * seeds a cut segment with the value just played, pipeline.cpp:193-196). */
const double* ga3c_ctx_last_values(ga3c_ctx* c);
/* Copy the last gradient and scalars to the host (blocking). */
int ga3c_ctx_read_grad(ga3c_ctx* c, float* dtheta, double* scalars);
/* Optional global-norm clip of the context gradient (nnet.cpp:281-289). */
int ga3c_clip_grad(ga3c_ctx* c);

/* Recompute the non-finite flag of grad_from's gradient (NULL = c; reset +
 * scan of all P values) on c's stream: after an in-place data-parallel
 * all-reduce the flag must describe the SUMMED gradient, so that every
 * replica rejects or applies the same step (nnet.cpp:299-301). */
int ga3c_check_grad(ga3c_ctx* c, ga3c_ctx* grad_from);
/* ------------------------------------------------------------ rmsprop */
/* SharedModel::apply pipeline.cpp:37-63 -> nnet::rmsprop_update
 * nnet.cpp:293-312: one non-centred RMSProp step on the LATEST parameters,
 * written out of place into a fresh slot and published as version+1.
 * dtheta: host gradient (P floats), or NULL to use the context gradient.
 * applied = 0 (status GA3C_NOT_APPLIED) when any gradient component is
 * non-finite; nothing changes then.  applied_on (nullable) = the version the
 * step was applied on top of. */
int ga3c_apply_rmsprop(ga3c_ctx* c, const float* dtheta, int* applied, uint64_t* applied_on);
/* nnet::rmsprop_update nnet.cpp:293-312 on a raw parameter vector of any
 * length n (no network layout): theta and g (host, n floats) are updated in
 * place on `device`; a non-finite dtheta leaves them unchanged and returns
 * GA3C_NOT_APPLIED with applied = 0.  Blocking. */
int ga3c_rmsprop_flat(const ga3c_hyper* hp, int device, size_t n, float* theta, float* g, const float* dtheta,
                      int* applied);
/* Stream-ordered device loop variant: updates the latest slot IN PLACE from
 * the context gradient, gated by the on-device non-finite flag; no host
 * synchronisation.  Only valid while no other thread reads the model. */
int ga3c_apply_rmsprop_dev(ga3c_ctx* c);
/* Device loop with several trainers in flight (GA3C's N_T trainer threads,
 * pipeline.cpp:241-306, each on its own context and stream): n extra
 * parameter slots, initialised from the latest snapshot and owned by the
 * caller (never recycled), into which the loop applies out of place --
 * update u reads slot ring[u % n] and writes ring[(u + 1) % n], so a
 * trainer still reading an older version is never overwritten. */
int ga3c_model_ring(ga3c_model* m, int n, int* slots_out);
/* One RMSProp step from src_slot into dst_slot with the gradient and
 * non-finite flag of context grad_from (NULL = c), stream-ordered on c's
 * stream; the caller orders grad_from's stream before it.  Capturable. */
int ga3c_apply_rmsprop_slots_dev(ga3c_ctx* c, const ga3c_ctx* grad_from, int src_slot, int dst_slot);
/* SMs this context's split-K plans try to fill (0 = all).  With N_T trainer contexts in
 * flight a share of the SMs per context costs less SM time per update
 * (fewer, longer CTAs) than a full wave each.  Results do not change
 * (every reduction is fixed-order for a given plan; parity tolerances hold
 * for any plan). */
int ga3c_ctx_set_sm_budget(ga3c_ctx* c, int sms);
/* Scheduling priority of the context's stream: 0 = the device's highest
 * (the default: a predictor's forward is on the agents' critical path),
 * level k = k steps lower (clamped to the lowest).  GA3C's trainers are
 * throughput work beside latency-bound predictions (pipeline.cpp:153-205
 * vs 241-306), so the native trainer pool and engine run their trainer
 * contexts one level below the predictors.  Call while the context is idle
 * and before capturing graphs on it (captured kernels keep the priority
 * they were captured at). */
int ga3c_ctx_set_priority(ga3c_ctx* c, int level);
/* Copy parameter slot src_slot's theta and rms state into dst_slot,
 * stream-ordered on c's stream (capturable): e.g. publish the last version of
 * a device loop to a predictor-only slot that the trainers never write, so
 * predictors and trainers run concurrently (GA3C, pipeline.hpp:87-91). */
int ga3c_copy_slot_dev(ga3c_ctx* c, int src_slot, int dst_slot);
/* ---------------------------------------- data parallel, fused over NVLink
 * One kernel per update replaces NCCL all-reduce(sum) + RMSProp on every
 * replica: rank r reduces shard r of every
 * rank's gradient over peer memory (fixed rank order), the non-finite reject
 * and the optional clip are decided globally, RMSProp runs on the shard and
 * theta' is stored into every rank's destination slot.  The rms state is
 * sharded (each replica maintains only its own shard of g).  Peer pointers
 * come from CUDA IPC (ga3c_ipc_*) or, for ranks that share a device, are the
 * raw device pointers.  Replaces the NCCL path of dp.py's dp_update. */
typedef struct ga3c_dp ga3c_dp;
/* ctas: CTAs per call (<= 148, identical on every rank; all must be
 * co-resident with the other ranks' calls). */
ga3c_dp* ga3c_dp_create(ga3c_model* m, int rank, int world, int ctas, int* status);
void ga3c_dp_destroy(ga3c_dp* dp);
/* This rank's signal block (device memory, to be mapped into every peer). */
void* ga3c_dp_signal(ga3c_dp* dp);
/* Synchronises the device; GA3C_CUDA_ERROR if any call of this dp timed out
 * waiting for a peer (the call then left its destination unreliable). */
int ga3c_dp_check(ga3c_dp* dp);
/* Device pointer of a parameter slot's theta (for the peers' destination list). */
int ga3c_model_slot_theta(ga3c_model* m, int slot, float** theta);
/* One fused update on c's stream: gradient of grad_from (NULL = c), source
 * and destination slots of this rank, and per-rank arrays (world entries,
 * index = rank) of gradient buffers, destination thetas and signal blocks as
 * mapped in this process.  Every rank must make the same sequence of calls. */
int ga3c_dp_apply(ga3c_ctx* c, ga3c_dp* dp, const ga3c_ctx* grad_from, int src_slot, int dst_slot,
                  float* const* peer_grads, float* const* peer_theta_dst, void* const* peer_signals);
/* CUDA IPC of library allocations (64-byte handles). */
int ga3c_ipc_get_handle(const void* dev_ptr, void* handle64);
int ga3c_ipc_open_handle(const void* handle64, void** dev_ptr);
int ga3c_ipc_close(void* dev_ptr);
/* On-device update counter of ga3c_apply_rmsprop_dev (blocking read). */
int ga3c_ctx_read_dev_version(ga3c_ctx* c, uint64_t* version);

/* ------------------------------------ data parallel through NCCL (§8e) */
/* in-place ncclAllReduce(sum) of
 * grad_from's gradient (NULL = c) over `nccl_comm` (an ncclComm_t) on c's
 * stream, then the non-finite flag recomputed on the sum (ga3c_check_grad),
 * so every replica applies or rejects the same step and stays bit-identical.
 * Follow with ga3c_clip_grad (if clipping) and the apply.  NCCL is loaded at
 * run time (libnccl.so.2; the copy already in the process if any):
 * GA3C_NCCL_ERROR when it is unavailable.  Capturable. */
int ga3c_allreduce_grads(ga3c_ctx* c, ga3c_ctx* grad_from, void* nccl_comm);
/* Communicator plumbing for callers without their own NCCL binding: rank 0
 * draws the 128-byte id, the caller broadcasts it, every rank inits. */
int ga3c_nccl_unique_id(void* id128);
int ga3c_nccl_comm_init(int world, const void* id128, int rank, int device, void** comm);
int ga3c_nccl_comm_destroy(void* comm);
int ga3c_nccl_version(int* version);
/* The model a context belongs to. */
ga3c_model* ga3c_ctx_model(ga3c_ctx* c);

/* ------------------------------------------------------------ returns */
/* returns::compute_returns returns.hpp:31 / returns.cpp:8-26, batched over
 * n_seg segments: segment s covers rewards[seg_offsets[s] .. seg_offsets[s+1]).
 * fp64 with the reference's operation order (bitwise).  Host buffers. */
int ga3c_compute_returns(ga3c_ctx* c, const double* rewards, const int32_t* seg_offsets,
                         int n_seg, const uint8_t* terminal, const double* bootstrap,
                         double gamma, double* out);
/* Device variant (async, no validation); d_out feeds ga3c_loss_grad_dev. */
int ga3c_compute_returns_dev(ga3c_ctx* c, const double* d_rewards, const int32_t* d_seg_offsets,
                             int n_seg, const uint8_t* d_terminal, const double* d_bootstrap,
                             double gamma, double* d_out);

/* Page-locked host memory (cudaMallocHost): copies between it and the
 * device are asynchronous DMA (the engine's predictor stages frames here). */
void* ga3c_host_alloc(size_t bytes, int* status);
void ga3c_host_free(void* p);

/* -------------------------------------------------------- frame store */
/* Device-resident 4-frame stacks.  The reference's
 * PredictionRequest carries the whole stacked state (pipeline.hpp:23-27);
 * here an agent sends only its NEWEST frame (in_h x in_w bytes) and the
 * store shifts it into that agent's stack on the device (channel 0 = oldest
 * frame, 3 = newest; an episode start -- reset or the agent's first push --
 * repeats the frame four times).  Each agent's last `history` stacked states
 * stay on the device, so training gathers its experiences from there instead
 * of copying them to the GPU a second time (the TrainingQueue's
 * Experience.state, returns.hpp:13-19).  Needs in_c == 4. */
typedef struct ga3c_frames ga3c_frames;
ga3c_frames* ga3c_frames_create(ga3c_model* m, int n_agents, int history, int* status);
void ga3c_frames_destroy(ga3c_frames* f);
/* Predictor call (predictor_loop pipeline.cpp:65-93 with the frame push):
 * push new_frames[n][in_h*in_w] for agents[n] (resets nullable), forward the
 * n new stacked states on snapshot `slot` (-1 = latest) and return pi / v as
 * in ga3c_forward_u8.  state_slots (nullable, n) receives where each new
 * state is stored -- the handle training uses. */
int ga3c_predict_frames(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                        const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots,
                        float* pi, float* v, uint64_t* version_used);
/* The same with pi as the device's fp64 softmax and V widened to fp64 (see
 * ga3c_forward64_u8): host-side qac::sample_index on these rows draws the
 * action the on-device sampler draws. */
int ga3c_predict_frames64(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                          const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots, double* pi,
                          double* v, uint64_t* version_used);
/* The same split in two: _async pushes the frames and enqueues the forward
 * and the copies of pi / V into the context's pinned stage, then returns
 * (state_slots are filled at once); ga3c_predict_collect64 waits for them
 * and copies them out.  One prediction may be in flight per context, and
 * until it is collected the context takes no other host-buffer call; the
 * caller keeps new_frames unchanged until then (page-locked frames are
 * copied asynchronously).  A predictor thread can so keep two contexts'
 * batches in flight (e.g. two agent groups).  After the frames' upload, the
 * device work of an _async call (stage upload, frame push, forward, sampling,
 * result download) is one CUDA graph captured per (snapshot slot, n, outputs,
 * store) on first use and replayed afterwards; a change of the context's SM
 * budget or priority drops its graphs. */
int ga3c_predict_frames64_async(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                                const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots);
int ga3c_predict_collect64(ga3c_ctx* c, double* pi, double* v, uint64_t* version_used);
/* As ga3c_predict_frames64_async, plus the agents' actions drawn on the
 * device: u[i] is agent i's uniform draw (qac::next_uniform), and
 * sample_kernel applies qac::sample_index (util.hpp:46-54) to the fp64
 * policy -- bitwise the action host-side sampling of the returned pi draws
 * (pipeline.cpp:172-173).  ga3c_predict_collect_act64 waits and copies out
 * actions, V and (pi != NULL) the fp64 policy; ga3c_predict_collect64 also
 * collects such a prediction (pi and V only). */
int ga3c_predict_frames_act64_async(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                                    const int32_t* agents, const uint8_t* resets, int n, const double* u,
                                    int32_t* state_slots);
int ga3c_predict_collect_act64(ga3c_ctx* c, int32_t* actions, double* v, double* pi, uint64_t* version_used);
/* Trainer call: as ga3c_loss_grad_segments_u8, with sample b's state read
 * from the store at (agents[b], state_slots[b]) on the device. */
int ga3c_train_frames(ga3c_ctx* c, int slot, ga3c_frames* f, const int32_t* agents,
                      const int32_t* state_slots, int B, const int32_t* actions, const double* rewards,
                      const int32_t* seg_offsets, int n_seg, const uint8_t* terminal,
                      const double* bootstrap, double gamma, int apply_clip, double* scalars,
                      double* returns_out);
/* Copy one stored stacked state to the host (tests, debugging). */
int ga3c_frames_read(ga3c_frames* f, int agent, int state_slot, uint8_t* state);

/* ------------------------------------------------------- trainer pool */
/* GA3C's TrainingQueue + trainer threads (pipeline.cpp:241-306) as a
 * component for hosts that run their own agents and predictors: n_threads
 * native trainers, each with its own context (SM budget `sms`, 0 = all),
 * take submitted segment batches in FIFO order and run ga3c_train_frames on
 * the latest snapshot + ga3c_apply_rmsprop (a non-finite gradient is
 * rejected and counted, nnet.cpp:299-301).  submit() copies its host
 * arrays (the ga3c_train_frames arguments) and blocks while queue_cap
 * batches are waiting; wait() returns once every submitted batch is applied
 * (or rejected), with the totals so far and the first error. */
typedef struct ga3c_trainer_pool ga3c_trainer_pool;
ga3c_trainer_pool* ga3c_trainer_pool_create(ga3c_model* m, ga3c_frames* f, int n_threads, int max_batch, int sms,
                                            int queue_cap, int* status);
int ga3c_trainer_pool_submit(ga3c_trainer_pool* p, const int32_t* agents, const int32_t* state_slots, int B,
                             const int32_t* actions, const double* rewards, const int32_t* seg_offsets, int n_seg,
                             const uint8_t* terminal, const double* bootstrap, double gamma);
/* n_batches submits in one call: batch i covers samples
 * [batch_off[i], batch_off[i+1]) of the concatenated per-sample arrays and
 * segments [seg_base[i], seg_base[i+1]) of terminal / bootstrap, whose
 * offsets (relative to the batch, each list starting at 0) are
 * seg_offsets[seg_base[i] + i .. seg_base[i+1] + i]. */
int ga3c_trainer_pool_submit_many(ga3c_trainer_pool* p, int n_batches, const int32_t* batch_off,
                                  const int32_t* seg_base, const int32_t* agents, const int32_t* state_slots,
                                  const int32_t* actions, const double* rewards, const int32_t* seg_offsets,
                                  const uint8_t* terminal, const double* bootstrap, double gamma);
int ga3c_trainer_pool_wait(ga3c_trainer_pool* p, long long* updates, long long* rejected);
const char* ga3c_trainer_pool_error(ga3c_trainer_pool* p);
void ga3c_trainer_pool_destroy(ga3c_trainer_pool* p);

/* ------------------------------------------------------ timing probe */
/* Kernel classes for the roofline probe. */
#define GA3C_K_NONE 0
#define GA3C_K_CONV_FWD 1
#define GA3C_K_FC_FWD 2
#define GA3C_K_HEADS 3
#define GA3C_K_LOSS_BWD 4
#define GA3C_K_WGRAD 5
#define GA3C_K_DGRAD 6
#define GA3C_K_SPLITK 7
#define GA3C_K_RMSPROP 8
#define GA3C_K_RETURNS 9
#define GA3C_K_SAMPLE 10
#define GA3C_K_OTHER 11
/* Bracket every subsequent launch of kernel class `tag` (trunk layer `layer`,
 * -1 = any) with CUDA events on the context stream (GA3C_K_NONE disables). */
int ga3c_ctx_time_kernel(ga3c_ctx* c, int tag, int layer);
/* Sum of the bracketed device durations since the last call (blocking). */
int ga3c_ctx_kernel_time(ga3c_ctx* c, double* total_ms, uint64_t* launches);
/* Bracket every launch (profiling): with ga3c_ctx_time_kernel(c, GA3C_K_ALL,
 * -1), ga3c_ctx_timeline returns up to `cap` launches since the last read:
 * start / end in ms relative to the first bracketed launch, kernel class,
 * trunk layer (-1 = none) and stream (0 = context stream, 1/2 = the side
 * streams of the backward DAG).  Blocking; resets the record. */
#define GA3C_K_ALL 12
int ga3c_ctx_timeline(ga3c_ctx* c, int cap, double* start_ms, double* end_ms, int* tags, int* layers,
                      int* streams, int* n);

/* ------------------------------------------------------- CUDA graphs */
/* Capture the device-resident calls issued on this context's stream between
 * begin and end (forward_dev / loss_grad_dev / apply_rmsprop_dev / ...) into
 * a CUDA graph; launch replays it.  Shapes and pointers are frozen at capture
 * time.  No host-synchronising call may be made while capturing. */
int ga3c_ctx_graph_begin(ga3c_ctx* c);
int ga3c_ctx_graph_end(ga3c_ctx* c, int* graph_id);
int ga3c_ctx_graph_launch(ga3c_ctx* c, int graph_id);

/* ----------------------------------------------------------- sampling */
/* qac::sample_index util.hpp:46-54 per row: the first a with u < sum_{<=a} pi
 * accumulated in fp64.  d_pi = NULL samples the context's last forward output
 * using its fp64 softmax; otherwise the fp32 rows of d_pi.  Device buffers,
 * async. */
int ga3c_sample_actions_dev(ga3c_ctx* c, const float* d_pi, const double* d_u, int B,
                            int n_actions, int32_t* d_actions, int action_stride);

/* ------------------------------------------------- host engine (C++) */
/* pipeline::run (pipeline.hpp:122) / reference::train_sync (reference.hpp:30)
 * of the B200 host engine (paper_1611_06256_b200/csrc/host): agent threads
 * on CPU environments, predictor threads batching the PredictionQueue into
 * device forwards, trainer threads coalescing the TrainingQueue into device
 * returns + loss/backward + RMSProp, the control thread with the annealer. */
typedef struct ga3c_pipeline_opts {
  ga3c_net_spec net;
  ga3c_hyper hyper;
  /* EnvSpec (envs.hpp): 0 bandit, 1 catch, 2 delay lab, 3 frame catch (84x84x4
   * u8), 4 synthetic frames (84x84x4 u8, delay-lab ballast) */
  int env_kind, n_contexts, env_actions, grid_size;
  long long step_delay_us;
  int episode_len, action_repeat;
  /* KnobConfig (knobs.hpp:9-19) */
  int n_agents, n_predictors, n_trainers, pred_batch_max, min_train_batch, train_queue_cap, pred_queue_cap;
  /* StopCondition: 0 = unset */
  long long max_updates;
  double max_seconds;
  double target_score;
  int has_target_score;
  unsigned long long seed;
  int anneal, anneal_batches;
  double epoch_s;
  int max_agents, max_predictors, max_trainers;
  double metrics_interval_s;
  int greedy, sync_after_submit, capture_trajectory, device;
  /* 1 = device frame store (frame envs): agents send their newest 84x84
   * frame, stacks and the TrainingQueue's states stay on the GPU
   * (ga3c_frames_*); 0 = whole states both ways, as the reference. */
  int device_frames;
  /* SM budgets of the trainer / predictor contexts (ga3c_ctx_set_sm_budget):
   * -1 = automatic (trainers 3/4 of the SMs and predictors 64 when several
   * trainers share the GPU, else all), 0 = all SMs, n = n SMs. */
  int trainer_sms, predictor_sms;
} ga3c_pipeline_opts;

typedef struct ga3c_run_report {
  long long total_updates, skipped_updates, total_predictions, total_episodes;
  double wall_time_s, avg_tps, avg_pps, avg_samples_per_s, mean_lag, final_rolling_score;
  long long experiences_produced, experiences_trained, experiences_dropped, experiences_left_queued;
  int final_n_agents, final_n_predictors, final_n_trainers, final_pred_batch_max, final_min_train_batch;
  unsigned long long final_version;
  int n_trajectory, n_anneal, n_frames;
  double last_frame_tps, last_frame_pps, last_frame_pred_batch_mean;
} ga3c_run_report;

typedef struct ga3c_anneal_entry {
  int n_agents, n_predictors, n_trainers, pred_batch_max, min_train_batch;
  double measured_tps;
  int accepted;
} ga3c_anneal_entry;

void ga3c_default_pipeline_opts(ga3c_pipeline_opts* o);
/* sync_trainer = 1 runs train_sync (zero lag, round-robin agents).  Output
 * arrays are nullable; capacities bound what is copied.  err receives the
 * std::invalid_argument / runtime message. */
int ga3c_pipeline_run(const ga3c_pipeline_opts* o, int sync_trainer, ga3c_run_report* r,
                      float* final_theta, float* trajectory, int traj_cap, double* episode_scores,
                      int scores_cap, ga3c_anneal_entry* anneal, int anneal_cap, char* err, int err_len);

#ifdef __cplusplus
}
#endif
#endif /* GA3C_H */
