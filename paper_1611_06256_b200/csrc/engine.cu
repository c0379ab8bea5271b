// engine.cu -- device engine and C ABI of libga3c_b200.so (include/ga3c.h).
//
// ga3c_model  = the device side of SharedModel (pipeline.hpp:92-111): a ring
//               of immutable parameter slots {theta, g, version}.  Readers pin
//               a slot; apply() writes the RMSProp step out of place into a
//               free slot and publishes it, so a forward pass never sees a torn
//               update (pipeline.hpp:87-91) and the step lands on the LATEST
//               parameters while the gradient came from an older snapshot
//               (pipeline.cpp:285-287 vs 43-48).
// ga3c_ctx    = one predictor/trainer thread: a CUDA stream plus the
//               activation/gradient workspace for up to max_batch states.
//
// Forward (nnet.cpp:91-119) is a chain of implicit-GEMM launches, one per
// trunk layer, then the fused FC-finalize + heads + softmax kernel.
// loss_and_gradients (nnet.cpp:201-291) re-runs that forward keeping the
// activations, then the fused loss/heads-backward kernel and, per trunk layer
// from the top, a weight-gradient GEMM (bias gradient folded in as a ones
// column) and an input-gradient kernel gated by the previous activation.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <type_traits>
#include <vector>

#include "ga3c.h"
#include "kernels.cuh"
#include "layout.hpp"
#include "tc_gemm.cuh"
#include "tc_wgrad.cuh"
#include "tc_pipe.cuh"
#include "tc_ws.cuh"
#include <cudaTypedefs.h>

#include "tc_bf16.cuh"
#include "tc_dgrad.cuh"
#include "tc_u8conv.cuh"
#include "tc_wgrad_band.cuh"
#include "dp_fused.cuh"
#include "pdl.cuh"

using namespace ga3c;

namespace {

constexpr int kNumSMs = 148;
constexpr std::size_t kPartFloats = std::size_t(32) << 20;  // split-K scratch per ctx (128 MB)
// The scratch is cut into regions so branches of the backward DAG that run
// concurrently never share one: 0 = FC forward partials, 1 + li = weight
// gradient of trunk layer li, kRegions - 1 = heads.
constexpr int kRegions = GA3C_MAX_CONV + GA3C_MAX_HIDDEN + 2;
constexpr std::size_t kRegionFloats = kPartFloats / kRegions / 64 * 64;  // 256 B aligned
constexpr int kMaxActions = 64;
constexpr std::size_t kStageBytes = std::size_t(1) << 20;

struct Slot {
  float* theta = nullptr;
  float* g = nullptr;
  std::uint64_t version = 0;
  int refs = 0;
  // written by an asynchronous apply still in flight: device readers wait on
  // `ready`, host readers synchronise on it
  cudaEvent_t ready = nullptr;
  bool pending = false;
};

// Fixed-capacity slot storage: a Slot never moves once published, so a
// thread holding a slot index may read its immutable fields (theta, g) while
// another thread appends a slot.  Appends happen under update_m + read_m; the
// count is published with release order after the slot is fully written.
// Mutable fields (version, refs, pending, ready) are read under read_m.
constexpr int kMaxSlots = 64;
class SlotTable {
 public:
  int size() const { return n_.load(std::memory_order_acquire); }
  Slot& operator[](int i) { return s_[i]; }
  // false when the table is full (the caller reports GA3C_OUT_OF_MEMORY)
  bool push_back(const Slot& x) {
    const int k = n_.load(std::memory_order_relaxed);
    if (k >= kMaxSlots) return false;
    s_[k] = x;
    n_.store(k + 1, std::memory_order_release);
    return true;
  }
  Slot* begin() { return s_; }
  Slot* end() { return s_ + size(); }

 private:
  Slot s_[kMaxSlots];
  std::atomic<int> n_{0};
};

}  // namespace

struct ga3c_model {
  ga3c_net_spec spec{};
  ga3c_hyper hp{};
  Layout lo;
  int device = 0;
  std::mutex read_m;    // guards slots[].refs / version / cur  (pipeline.cpp:22-25)
  std::mutex update_m;  // serializes writers                   (pipeline.cpp:40)
  SlotTable slots;
  int cur = 0;
  // completion of the last asynchronous apply: the next writer orders after it
  cudaEvent_t apply_done = nullptr;
  bool apply_pending = false;
  std::mutex err_m;
  std::string last_error;
  void set_error(const std::string& e) {
    std::lock_guard<std::mutex> lk(err_m);
    last_error = e;
  }
};

struct ga3c_ctx {
  ga3c_model* m = nullptr;
  cudaStream_t stream = nullptr;
  // Kernels go to `cur`: the context stream, or a side stream while an
  // independent branch of the backward DAG (a weight gradient) is issued.
  cudaStream_t cur = nullptr;
  cudaStream_t side[2] = {};
  cudaEvent_t evs[16] = {};
  int ev_next = 0;
  int max_batch = 0;
  int sms = 0;  // SMs a split-K plan fills (ga3c_ctx_set_sm_budget; 0 = all)
  void* d_in = nullptr;
  float* act[GA3C_MAX_CONV + GA3C_MAX_HIDDEN] = {};
  float* dout[GA3C_MAX_CONV + GA3C_MAX_HIDDEN] = {};  // per-layer output gradient (backward DAG)
  float* hin = nullptr;  // f32 copy of a raw input feeding the heads directly
  float* pi32 = nullptr;
  double* pi64 = nullptr;
  float* v = nullptr;
  double* v64 = nullptr;
  float* dhead = nullptr;
  float* dhT = nullptr;  // transposed head-input gradient [D][ldT] (FC dgrad operand)
  int ldT = 0;
  double* scal = nullptr;
  double* scal_sum = nullptr;
  int32_t* d_actions = nullptr;
  double* d_rets = nullptr;
  float* grad = nullptr;
  int* flag = nullptr;  // control words: [0] non-finite flag, [1] heads-kernel ticket
  unsigned long long* dev_version = nullptr;
  float* part = nullptr;
  double* clip_part = nullptr;
  // returns / host staging
  double* r_rew = nullptr;
  int32_t* r_off = nullptr;
  uint8_t* r_term = nullptr;
  double* r_boot = nullptr;
  double* r_out = nullptr;
  std::size_t r_cap = 0, r_seg_cap = 0;
  int* h_flag = nullptr;  // pinned
  // non-finite flag of this context's last gradient, read back by the
  // host-buffer gradient calls (-1 = unknown: apply must read it itself)
  int grad_flag = -1;
  // staging for the host-buffer calls' small inputs and outputs: packed into
  // pinned memory and moved with ONE async copy each way (pageable
  // cudaMemcpyAsync is synchronous and costs microseconds per call)
  uint8_t* h_stage = nullptr;  // pinned, kStageBytes
  uint8_t* d_stage = nullptr;  // device, kStageBytes
  std::size_t stage_bytes = 0;
  int32_t* f_idx = nullptr;  // frame-store index staging
  std::size_t f_idx_cap = 0;
  std::uint64_t launches = 0;
  std::string last_error;
  // kernel timing probe (ga3c_ctx_time_kernel)
  int timed_tag = 0, timed_layer = -1;
  std::vector<cudaEvent_t> events;
  std::size_t ev_used = 0;
  std::vector<int> ev_meta;  // per bracketed launch: tag | layer << 8 | stream << 16
  // an asynchronous frame-store prediction in flight (ga3c_predict_frames64_async):
  // its outputs land in the pinned stage, the snapshot stays pinned until collected
  struct {
    bool active = false;
    const double* h_pi = nullptr;
    const double* h_v = nullptr;
    const int32_t* h_act = nullptr;  // device-sampled actions (ga3c_predict_frames_act64_async)
    int n = 0, A = 0, slot = -1;
    bool pinned = false;
    std::uint64_t ver = 0;
    cudaEvent_t ev = nullptr;
  } pend;
  // captured CUDA graphs of device-resident step sequences
  std::vector<cudaGraphExec_t> graphs;
  // ga3c_train_frames' device work (stage upload -> gather -> returns ->
  // loss/backward -> result download) captured once per (slot, B, segments,
  // outputs) and replayed: one launch per call instead of ~20 API calls
  struct TfKey {
    int slot, B, n_seg, flags;
    const void* ring;
    bool operator<(const TfKey& o) const {
      return std::tie(slot, B, n_seg, flags, ring) < std::tie(o.slot, o.B, o.n_seg, o.flags, o.ring);
    }
  };
  std::map<TfKey, cudaGraphExec_t> tf_graphs;
  bool capturing = false;
};

struct ga3c_frames {
  ga3c_model* m = nullptr;
  int n_agents = 0, history = 0;
  std::size_t frame_px = 0;   // bytes of one frame (in_h * in_w)
  uint8_t* ring = nullptr;    // [agent][history][in_h][in_w][4] u8 stacked states
  std::mutex mu;              // guards count (pushes per agent)
  std::vector<long long> count;
};

namespace {

#define GA3C_CUDA(call)                                                               \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      set_err(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
      return GA3C_CUDA_ERROR;                                                         \
    }                                                                                 \
  } while (0)

thread_local std::string g_tls_error;



// Every kernel goes out with programmatic stream serialization (pdl.cuh).
template <typename... KArgs, typename... Args>
void pdl_launch(cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// The same with a (cx, cy, cz) thread-block cluster.
template <typename... KArgs, typename... Args>
void pdl_launch_cluster(cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                        dim3 cluster, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cluster.x;
  at[1].val.clusterDim.y = cluster.y;
  at[1].val.clusterDim.z = cluster.z;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// --------------------------------------------------------------- GEMMs

struct SplitPlan {
  int splits = 1;
  int k_chunk = 0;
};

// Packs small host inputs into the context's pinned stage; flush() moves them
// to the device stage with one async copy.  put() returns the device address
// of the packed copy (nullptr when the stage is full: the caller falls back
// to a direct copy).  Outputs: take() reserves pinned space a D2H lands in.
struct Stager {
  ga3c_ctx* c;
  std::size_t off = 0;
  template <typename T>
  T* put(const T* src, std::size_t n) {
    const std::size_t b = n * sizeof(T);
    const std::size_t o = (off + 15) & ~static_cast<std::size_t>(15);
    if (o + b > c->stage_bytes) return nullptr;
    if (b) std::memcpy(c->h_stage + o, src, b);
    off = o + b;
    return reinterpret_cast<T*>(c->d_stage + o);
  }
  bool flush() {
    return off == 0 || cudaMemcpyAsync(c->d_stage, c->h_stage, off, cudaMemcpyHostToDevice, c->stream) == cudaSuccess;
  }
  // pinned host space for outputs, after everything put() so far
  template <typename T>
  T* take(std::size_t n) {
    const std::size_t o = (off + 15) & ~static_cast<std::size_t>(15);
    if (o + n * sizeof(T) > c->stage_bytes) return nullptr;
    off = o + n * sizeof(T);
    return reinterpret_cast<T*>(c->h_stage + o);
  }
};

int split_sms(const ga3c_ctx* c);

SplitPlan plan_splits(const ga3c_ctx* c, int M, int N, int K, bool allow_split) {
  SplitPlan p;
  const int tiles = ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
  int s = 1;
  if (allow_split) {
    s = std::max(1, (2 * split_sms(c) + tiles - 1) / tiles);
    s = std::min(s, std::max(1, K / 128));
    while (s > 1 && static_cast<std::size_t>(s) * M * N > kRegionFloats) --s;
  }
  int kc = (K + s - 1) / s;
  kc = ((kc + kBK - 1) / kBK) * kBK;
  if (kc <= 0) kc = kBK;
  p.k_chunk = kc;
  p.splits = std::max(1, (K + kc - 1) / kc);
  return p;
}

float* region(ga3c_ctx* c, int r) { return c->part + static_cast<std::size_t>(r) * kRegionFloats; }

// Branches of the backward DAG: fork() makes `s` wait for everything issued
// on the context stream so far and directs launches to it; join() makes the
// context stream wait for `s` and directs launches back.  Both are plain
// event edges, so they are captured into CUDA graphs as graph dependencies.
// (The design alternatives measured in round 1 -- serial backward, no side
// stream priorities, no cluster split-K, deep-only rings, ... -- are recorded
// with their numbers in DESIGN.md §5; the library builds only the measured
// best path.  It reads no environment variables.)
//
// SMs a split-K plan tries to fill (ga3c_ctx_set_sm_budget, default all
// 148): with several trainer contexts in flight, fewer and longer CTAs per
// kernel cost less SM time than one full wave each.
int split_sms(const ga3c_ctx* c) { return c && c->sms > 0 ? c->sms : kNumSMs; }
// Ring-depth cap (pipe::ring_depth) for a tensor-core launch whose CTAs
// each stream `n` k-chunks: no deeper than n; at most ~112 KB (two CTAs per
// SM) for multi-wave grids and for contexts sharing the GPU with other
// contexts (an SM budget below all SMs); otherwise as deep as fits.
int ring_cap(const ga3c_ctx* c, int n, long long ctas) {
  if (n <= 2) return 2;
  if (n == 3) return 3;
  return (ctas > kNumSMs || split_sms(c) < kNumSMs) ? 1 : 0;
}

// Raise a kernel's dynamic shared memory limit once per instantiation and
// device (the attribute is per device; a process may drive models on several
// devices).  Concurrent first launches may both set it, which is harmless;
// the bit is published only after the attribute is set.
void smem_once(std::atomic<unsigned long long>& done, const void* kern, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_acq_rel);
}
#define GA3C_SMEM_ONCE(kern, bytes)                         \
  static std::atomic<unsigned long long> smem_done_{0};     \
  smem_once(smem_done_, reinterpret_cast<const void*>(kern), static_cast<int>(bytes))

#define GA3C_CAP_SWITCH(cap, F) \
  switch (cap) {                \
    case 1: F(1); break;        \
    case 2: F(2); break;        \
    case 3: F(3); break;        \
    default: F(0); break;       \
  }

// SMs a cluster split-K plan (conv forward, FC input gradient) targets: the
// context's budget when it has the whole GPU, half of it when it shares the
// GPU with other trainers (N_T = 3: 0.25 / 0.5 / 2 x the budget measured
// slower than 1 x; re-swept at N_T = 6, DNN A, two runs each: 0.25 x
// 1.433-1.438M, 0.4 x 1.452-1.453M, 0.5 x 1.447-1.456M, 0.6 x 1.365-1.368M,
// 0.75 x 1.301M, 1 x 1.392-1.395M, 1.5 x 1.393M samples/s -- conv2 forward
// and FC input gradient at 2-way splits instead of 4).
int cluster_sms(const ga3c_ctx* c) {
  const int b = split_sms(c);
  return std::max(1, b >= kNumSMs ? b : b / 2);
}

void fork_to(ga3c_ctx* c, cudaStream_t s) {
  cudaEvent_t e = c->evs[c->ev_next++ & 15];
  cudaEventRecord(e, c->stream);
  cudaStreamWaitEvent(s, e, 0);
  c->cur = s;
}

void join_from(ga3c_ctx* c, cudaStream_t s) {
  cudaEvent_t e = c->evs[c->ev_next++ & 15];
  cudaEventRecord(e, s);
  cudaStreamWaitEvent(c->stream, e, 0);
  c->cur = c->stream;
}

// Brackets one launch with CUDA events when (tag, layer) is the probed kernel
// class; always counts the launch.
struct Launch {
  ga3c_ctx* c;
  bool on;
  bool ext = false;
  Launch(ga3c_ctx* c_, int tag, int layer) : c(c_) {
    on = c->timed_tag == GA3C_K_ALL ||
         (c->timed_tag == tag && (c->timed_layer < 0 || c->timed_layer == layer));
    if (on) {
      while (c->events.size() < c->ev_used + 2) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->events.push_back(e);
      }
      const int sid = c->cur == c->stream ? 0 : (c->cur == c->side[0] ? 1 : 2);
      c->ev_meta.resize(c->ev_used / 2 + 1);
      c->ev_meta[c->ev_used / 2] = tag | ((layer + 1) << 8) | (sid << 16);
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(c->cur, &cs);
      ext = cs == cudaStreamCaptureStatusActive;  // captured: an event-record node replayed with the graph
      cudaEventRecordWithFlags(c->events[c->ev_used], c->cur, ext ? cudaEventRecordExternal : cudaEventRecordDefault);
    }
  }
  ~Launch() {
    if (on) {
      cudaEventRecordWithFlags(c->events[c->ev_used + 1], c->cur, ext ? cudaEventRecordExternal : cudaEventRecordDefault);
      c->ev_used += 2;
    }
    c->launches++;
  }
};

template <class LA, class LB, class Epi>
void launch_gemm(ga3c_ctx* c, int tag, int layer, const LA& la, const LB& lb, const Epi& epi, int M,
                 int N, int K, const SplitPlan& p) {
  dim3 grid((N + kBN - 1) / kBN, (M + kBM - 1) / kBM, p.splits);
  Launch l(c, tag, layer);
  pdl_launch(c->cur, gemm_simt_kernel<LA, LB, Epi>, dim3(grid), dim3(kThreads), 0, la, lb, epi, M, N, K, p.k_chunk);
}

// ------------------------------------------------------ tensor-core GEMMs

template <typename TA, typename TB, int BN, int MODE, int CAP, bool TMA>
void tc_launch_v(ga3c_ctx* c, int tag, int layer, const Seg& A, const Seg& B, int M, int N, int K, int splits,
                 int kc, const TcEpiArgs& epi, const TmaConv& tm) {
  using S = ws::KKShape<TA, TB, BN, CAP>;
  auto kern = ws::tc_kk_ws_kernel<TA, TB, BN, MODE, CAP, TMA>;
  GA3C_SMEM_ONCE(kern, S::SMEM);
  dim3 grid((M + 127) / 128, splits, (N + BN - 1) / BN);
  Launch l(c, tag, layer);
  if (MODE == TC_EPI_BIAS_RELU && splits > 1)  // split-K reduced inside a cluster
    pdl_launch_cluster(c->cur, kern, dim3(grid), dim3(ws::kThreads), S::SMEM, dim3(1, splits, 1), A, B, M, N, K,
                       kc, epi, tm);
  else
    pdl_launch(c->cur, kern, dim3(grid), dim3(ws::kThreads), S::SMEM, A, B, M, N, K, kc, epi, tm);
}

template <typename TA, typename TB, int BN, int MODE, bool TMA>
void tc_launch(ga3c_ctx* c, int tag, int layer, const Seg& A, const Seg& B, int M, int N, int K, int splits,
               int kc, const TcEpiArgs& epi, const TmaConv& tm) {
  const long long ctas = static_cast<long long>((M + 127) / 128) * splits * ((N + BN - 1) / BN);
  const int cap = ring_cap(c, (std::min(kc, K) + 31) / 32, ctas);
#define GA3C_F(C) tc_launch_v<TA, TB, BN, MODE, C, TMA>(c, tag, layer, A, B, M, N, K, splits, kc, epi, tm)
  GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
}

template <typename TA, typename TB, int MODE, bool TMA = false>
void tc_dispatch(ga3c_ctx* c, int tag, int layer, int bn, const Seg& A, const Seg& B, int M, int N,
                 int K, int splits, int kc, const TcEpiArgs& epi, const TmaConv& tm = TmaConv{}) {
  switch (bn) {
    case 16: tc_launch<TA, TB, 16, MODE, TMA>(c, tag, layer, A, B, M, N, K, splits, kc, epi, tm); break;
    case 32: tc_launch<TA, TB, 32, MODE, TMA>(c, tag, layer, A, B, M, N, K, splits, kc, epi, tm); break;
    case 64: tc_launch<TA, TB, 64, MODE, TMA>(c, tag, layer, A, B, M, N, K, splits, kc, epi, tm); break;
    default: tc_launch<TA, TB, 128, MODE, TMA>(c, tag, layer, A, B, M, N, K, splits, kc, epi, tm); break;
  }
}

// Tensor maps of a TMA-staged conv forward (TmaConv): im2col over the NHWC
// fp32 input [B][IH][IW][Cin] and tiles of the OHWI weights.  False when the
// driver entry points are missing or the geometry is outside what the TMA
// im2col mode encodes (the cp.async gather path is used then).
bool conv_tma_maps(const Layer& L, const float* x, const float* w, int B, int bn, TmaConv* tm) {
  static PFN_cuTensorMapEncodeIm2col enc_im2col = nullptr;
  static PFN_cuTensorMapEncodeTiled enc_tiled = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col>(f);
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(f);
  });
  if (!enc_im2col || !enc_tiled) return false;
  if (L.cin % 32 != 0 || L.k - 1 > 127 || L.stride > 8 || (reinterpret_cast<uintptr_t>(x) % 16) != 0 ||
      (reinterpret_cast<uintptr_t>(w) % 16) != 0)
    return false;
  const cuuint64_t gdim[4] = {static_cast<cuuint64_t>(L.cin), static_cast<cuuint64_t>(L.iw),
                              static_cast<cuuint64_t>(L.ih), static_cast<cuuint64_t>(B)};
  const cuuint64_t gstride[3] = {static_cast<cuuint64_t>(L.cin) * 4, static_cast<cuuint64_t>(L.iw) * L.cin * 4,
                                 static_cast<cuuint64_t>(L.ih) * L.iw * L.cin * 4};
  const int lower[2] = {0, 0};
  const int upper[2] = {-(L.k - 1), -(L.k - 1)};  // VALID: the window corner spans [0, I - k]
  const cuuint32_t estride[4] = {1, static_cast<cuuint32_t>(L.stride), static_cast<cuuint32_t>(L.stride), 1};
  if (enc_im2col(&tm->a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), gdim, gstride, lower, upper, 32,
                 128, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const cuuint64_t wdim[2] = {static_cast<cuuint64_t>(L.in), static_cast<cuuint64_t>(L.cout)};
  const cuuint64_t wstride[1] = {static_cast<cuuint64_t>(L.in) * 4};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(bn)};
  const cuuint32_t one[2] = {1, 1};
  if (enc_tiled(&tm->b, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(w), wdim, wstride, box, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  tm->cin = L.cin;
  tm->k = L.k;
  tm->stride = L.stride;
  return true;
}

int tc_bn(int n) {  // N tile; 2*BN (hi|lo concatenated) must fit one MMA (<= 256)
  int b = 16;
  while (b < n && b < 128) b *= 2;
  return b;
}

// Every (row, 32-chunk) run must be 16-byte aligned (fp32: 4 elements) or
// 4-byte aligned (u8), and element offsets must fit the kernel's int32 math.
bool seg_ok(const Seg& s, int rows_total) {
  return s.rowlen % 32 == 0 && s.bstride % 4 == 0 && s.rs_y % 4 == 0 && s.rs_x % 4 == 0 &&
         s.kstride % 4 == 0 && (reinterpret_cast<uintptr_t>(s.p) % 16) == 0 &&
         static_cast<double>(s.bstride) * (rows_total / std::max(1, s.P) + 1) < 2.0e9;
}

template <typename T>
Seg conv_seg(const Layer& L, const void* x, long long bstride) {
  Seg s;
  s.p = x;
  s.bstride = bstride > 0 ? bstride : static_cast<long long>(L.ih) * L.iw * L.cin;
  s.P = L.oh * L.ow;
  s.ow = L.ow;
  s.rs_y = L.stride * L.iw * L.cin;
  s.rs_x = L.stride * L.cin;
  s.rowlen = L.k * L.cin;
  s.kstride = L.iw * L.cin;
  s.rows = 0;
  return s;
}

Seg dense_seg(const void* p, int rows, long long ld, int K, bool u8) {
  Seg s;
  s.p = p;
  s.bstride = ld;
  s.P = 1;
  s.ow = 1;
  s.rs_y = 0;
  s.rs_x = 0;
  s.rowlen = K;
  s.kstride = 0;
  s.rows = rows;
  (void)u8;
  return s;
}

template <typename T>
Im2col<T> im2col_of(const Layer& L, const void* x, long long bstride) {
  Im2col<T> g;
  g.bstride = bstride > 0 ? bstride : static_cast<long long>(L.ih) * L.iw * L.cin;
  g.p = static_cast<const T*>(x);
  g.ih = L.ih;
  g.iw = L.iw;
  g.cin = L.cin;
  g.stride = L.stride;
  g.ow = L.ow;
  g.P = L.oh * L.ow;
  g.rowlen = L.k * L.cin;
  return g;
}

template <int BN, int CAP>
void u8_conv_launch(ga3c_ctx* c, int li, const Seg& A, const Seg& W, int M, int N, int K, int ks, int kc,
                    const TcEpiArgs& e) {
  using S = bf::U8Shape<BN>;
  constexpr int NS = pipe::ring_depth(CAP, S::STAGE);
  constexpr int SMEM = NS * S::STAGE + 1024;
  auto kern = bf::tc_u8_fwd_kernel<BN, CAP>;
  GA3C_SMEM_ONCE(kern, SMEM);
  dim3 grid((M + 127) / 128, ks, (N + BN - 1) / BN);
  Launch l(c, GA3C_K_CONV_FWD, li);
  if (ks > 1)
    pdl_launch_cluster(c->cur, kern, grid, dim3(bf::kThreads), SMEM, dim3(1, ks, 1), A, W, M, N, K, kc, e);
  else
    pdl_launch(c->cur, kern, grid, dim3(bf::kThreads), SMEM, A, W, M, N, K, kc, e);
}

// Conv on raw u8 frames through the exact bf16 split (tc_bf16.cuh).
// Persistent weight-stationary u8 conv (tc_u8conv.cuh); false when the
// geometry is outside what it handles.
template <int BN>
void u8_persist_launch(ga3c_ctx* c, int li, const u8c::ConvArgs& a, dim3 grid) {
  using S = u8c::Shape<BN>;
  auto kern = u8c::tc_u8conv_kernel<BN>;
  GA3C_SMEM_ONCE(kern, S::SMEM);
  Launch l(c, GA3C_K_CONV_FWD, li);
  pdl_launch(c->cur, kern, grid, dim3(u8c::kThreads), S::SMEM, a);
}

bool u8_conv_persistent(ga3c_ctx* c, int li, const Layer& L, const float* theta, const uint8_t* x,
                        long long bstride, float* out, int B) {
  const int P = L.oh * L.ow;
  const int rowb = L.iw * L.cin;
  if (P < 128 || L.cin % 4 != 0 || rowb % 16 != 0 || L.in % 128 != 0 || L.in > u8c::kMaxK ||
      (L.k * L.cin) % 16 != 0 || L.cout > 32 || L.cout % 4 != 0 || L.w_off % 4 != 0 || bstride % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(x) % 16) != 0)
    return false;
  // footprint bound: at most floor(127/ow)+2 output rows over at most two frames
  const int span = 127 / L.ow;
  const int rows = std::max((span + 1) * L.stride + L.k, span * L.stride + 2 * L.k);
  // one tile per CTA gains nothing from persistence, and its 180 KB of smem
  // would keep concurrent kernels off the SM: small grids take tc_bf16.cuh --
  // except in a context sharing the GPU, where ~4 tiles per CTA on a quarter
  // as many CTAs beat one tile per CTA (DNN A trainers, B = 40, 125 tiles,
  // two runs each at N_T = 6: 16 CTAs 1.462M, 24 1.475-1.478M, 32
  // 1.476-1.478M, 40 1.417-1.463M, 48 1.450-1.453M, 64 1.425M, tc_bf16.cuh's
  // 125 CTAs 1.451-1.454M samples/s)
  const int tiles = (B * P + 127) / 128;
  const bool shared = split_sms(c) < kNumSMs;
  if (tiles < 2 * kNumSMs && !(shared && tiles >= 64)) return false;
  const int fp_bytes = ((rows * rowb + 16) + 127) / 128 * 128;
  const int fp_stages = std::min(u8c::kFpMaxStages, u8c::kFpRegion / fp_bytes);
  if (fp_stages < 2) return false;
  u8c::ConvArgs a{x, bstride, theta + L.w_off, theta + L.b_off, out, L.cout, B, L.ih, L.iw, L.cin, L.k,
                  L.stride, L.oh, L.ow, L.cout, L.in, (B * P + 127) / 128, fp_bytes, fp_stages};
  const int bn = L.cout <= 16 ? 16 : 32;
  const int ctas = std::min({tiles, split_sms(c), shared ? std::max(1, tiles / 4) : kNumSMs});
  dim3 grid(static_cast<unsigned>(ctas), (L.cout + bn - 1) / bn, 1);
  if (bn == 16)
    u8_persist_launch<16>(c, li, a, grid);
  else
    u8_persist_launch<32>(c, li, a, grid);
  return true;
}

bool u8_conv_forward(ga3c_ctx* c, int li, const Layer& L, const float* theta, const Seg& A, float* out, int B) {
  if (u8_conv_persistent(c, li, L, theta, static_cast<const uint8_t*>(A.p), A.bstride, out, B))
    return true;
  const int bn = tc_bn(L.cout);
  if (L.in % 64 != 0 || (L.k * L.cin) % 32 != 0 || bn > 64 || L.cout % 4 != 0 || L.w_off % 4 != 0 ||
      A.rowlen % 32 != 0)
    return false;
  Seg W = dense_seg(theta + L.w_off, L.cout, L.in, L.in, false);
  TcEpiArgs e{theta + L.b_off, out, L.cout};
  const int M = B * L.pixels();
  const int tiles = ((M + 127) / 128) * ((L.cout + bn - 1) / bn);
  const int chunks = L.in / 64;
  int ks = std::max(1, std::min({8, chunks, cluster_sms(c) / std::max(1, tiles)}));
  const int kc = ((chunks + ks - 1) / ks) * 64;
  ks = (L.in + kc - 1) / kc;
  const int cap = ring_cap(c, (std::min(kc, L.in) + 63) / 64, static_cast<long long>(tiles) * ks);
  switch (bn) {
    case 16: {
#define GA3C_F(C) u8_conv_launch<16, C>(c, li, A, W, M, L.cout, L.in, ks, kc, e)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
    case 32: {
#define GA3C_F(C) u8_conv_launch<32, C>(c, li, A, W, M, L.cout, L.in, ks, kc, e)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
    default: {
#define GA3C_F(C) u8_conv_launch<64, C>(c, li, A, W, M, L.cout, L.in, ks, kc, e)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
  }
  return true;
}

template <typename T>
void conv_forward(ga3c_ctx* c, int li, const Layer& L, const float* theta, const void* x, float* out,
                  int B, long long in_stride) {
  if constexpr (sizeof(T) == 1) {
    Seg A = conv_seg<T>(L, x, in_stride);
    A.rows = B * L.pixels();
    if (seg_ok(A, A.rows) && u8_conv_forward(c, li, L, theta, A, out, B)) return;
  }
  {
    Seg A = conv_seg<T>(L, x, in_stride);
    A.rows = B * L.pixels();
    Seg W = dense_seg(theta + L.w_off, L.cout, L.in, L.in, false);
    if (seg_ok(A, A.rows) && L.in % 32 == 0 && L.cout <= 128 && L.cout % 4 == 0 && (L.w_off % 4) == 0) {
      TcEpiArgs e{theta + L.b_off, out, L.cout};
      const int M = B * L.pixels();
      const int bn = tc_bn(L.cout);
      // Fewer tiles than SMs: split K over a cluster of up to 8 CTAs whose
      // partial tiles are summed through DSMEM in the epilogue.
      const int tiles = ((M + 127) / 128) * ((L.cout + bn - 1) / bn);
      const int chunks = L.in / 32;
      int ks = std::max(1, std::min({8, chunks, cluster_sms(c) / std::max(1, tiles)}));
      const int kc = ((chunks + ks - 1) / ks) * 32;
      ks = (L.in + kc - 1) / kc;
      if constexpr (sizeof(T) == 4) {
        // fp32 input with whole 32-channel taps: TMA-staged operands
        TmaConv tm;
        if (in_stride <= 0 && conv_tma_maps(L, static_cast<const float*>(x), theta + L.w_off, B, bn, &tm)) {
          tc_dispatch<float, float, TC_EPI_BIAS_RELU, true>(c, GA3C_K_CONV_FWD, li, bn, A, W, M, L.cout, L.in, ks,
                                                            kc, e, tm);
          return;
        }
      }
      tc_dispatch<T, float, TC_EPI_BIAS_RELU>(c, GA3C_K_CONV_FWD, li, bn, A, W, M, L.cout, L.in, ks, kc, e);
      return;
    }
  }
  Im2colA<T> a;
  static_cast<Im2col<T>&>(a) = im2col_of<T>(L, x, in_stride);
  DenseK w{theta + L.w_off, L.in};
  const int M = B * L.pixels();
  launch_gemm(c, GA3C_K_CONV_FWD, li, a, w, EpiBiasRelu{out, theta + L.b_off, L.cout}, M, L.cout,
              L.in, plan_splits(c, M, L.cout, L.in, false));
}

// FC forward.  If `keep_partials` the split-K partials are left in c->part for
// the fused heads kernel; returns the number of splits used.
template <typename T>
int fc_forward(ga3c_ctx* c, int li, const Layer& L, const float* theta, const void* x, float* out,
               int B, bool keep_partials, long long in_stride) {
  const long long ld = in_stride > 0 ? in_stride : L.in;
  {
    Seg X = dense_seg(x, B, ld, L.in, sizeof(T) == 1);
    Seg W = dense_seg(theta + L.w_off, L.out, L.in, L.in, false);
    if (seg_ok(X, B) && seg_ok(W, L.out) && (L.w_off % 4) == 0 && L.out % 4 == 0) {
      // swap-AB: the 128-row MMA tile runs over output units, batch is N
      const int bn = tc_bn(B);
      const int tiles = ((L.out + 127) / 128) * ((B + bn - 1) / bn);
      const int chunks = L.in / 32;
      int splits = std::max(1, std::min(chunks, split_sms(c) / std::max(1, tiles)));
      while (splits > 1 && static_cast<std::size_t>(splits) * B * L.out > kRegionFloats) --splits;
      const int kc = ((chunks + splits - 1) / splits) * 32;
      splits = (L.in + kc - 1) / kc;
      TcEpiArgs e{nullptr, region(c, 0), L.out};
      tc_dispatch<float, T, TC_EPI_PART_T>(c, GA3C_K_FC_FWD, li, bn, W, X, L.out, B, L.in, splits, kc, e);
      if (!keep_partials) {
        const std::size_t n = static_cast<std::size_t>(B) * L.out;
        Launch l(c, GA3C_K_SPLITK, li);
        pdl_launch(c->cur, splitk_bias_relu_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, 
            region(c, 0), splits, B, L.out, theta + L.b_off, out);
      }
      return splits;
    }
  }
  DenseKIn<T> a{static_cast<const T*>(x), static_cast<int>(ld)};
  DenseK w{theta + L.w_off, L.in};
  const SplitPlan p = plan_splits(c, B, L.out, L.in, true);
  if (keep_partials || p.splits > 1) {
    launch_gemm(c, GA3C_K_FC_FWD, li, a, w, EpiPartial{region(c, 0), B, L.out}, B, L.out, L.in, p);
    if (!keep_partials) {
      const std::size_t n = static_cast<std::size_t>(B) * L.out;
      Launch l(c, GA3C_K_SPLITK, li);
      pdl_launch(c->cur, splitk_bias_relu_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, 
          region(c, 0), p.splits, B, L.out, theta + L.b_off, out);
    }
  } else {
    launch_gemm(c, GA3C_K_FC_FWD, li, a, w, EpiBiasRelu{out, theta + L.b_off, L.out}, B, L.out, L.in, p);
  }
  return p.splits;
}

void launch_splitk_grad(ga3c_ctx* c, int li, int splits, int M, int N, const GradMap& gm, float* part) {
  const std::size_t n = static_cast<std::size_t>(M) * N;
  Launch l(c, GA3C_K_SPLITK, li);
  if (splits > 16)
    pdl_launch(c->cur, splitk_grad8_kernel, dim3((unsigned)((n + 31) / 32)), dim3(256), 0, part, splits, M, N, gm);
  else
    pdl_launch(c->cur, splitk_grad_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, part, splits, M, N, gm);
}

// Weight-gradient GEMM [M rows][N = Kw+1] (+ reduction) into dtheta.
template <class LA, class LB>
void wgrad_gemm(ga3c_ctx* c, int li, const LA& la, const LB& lb, const GradMap& gm, int M, int N,
                int K, float* part) {
  const SplitPlan p = plan_splits(c, M, N, K, true);
  if (p.splits == 1) {
    launch_gemm(c, GA3C_K_WGRAD, li, la, lb, EpiGrad{gm}, M, N, K, p);
  } else {
    launch_gemm(c, GA3C_K_WGRAD, li, la, lb, EpiPartial{part, M, N}, M, N, K, p);
    launch_splitk_grad(c, li, p.splits, M, N, gm, part);
  }
}

template <typename TX, int BN, int CAP>
void wgrad_tc_launch_v(ga3c_ctx* c, int li, const WgradArgs& a, dim3 grid, int tag) {
  using S = ws::MNShape<TX, BN, CAP>;
  auto kern = ws::tc_mn_ws_kernel<TX, BN, CAP>;
  GA3C_SMEM_ONCE(kern, S::SMEM);
  Launch l(c, tag, li);
  if ((a.mode == 1 || a.cluster) && grid.y > 1)  // split-K reduced inside a cluster
    pdl_launch_cluster(c->cur, kern, dim3(grid), dim3(ws::kThreads), S::SMEM, dim3(1, grid.y, 1), a);
  else
    pdl_launch(c->cur, kern, dim3(grid), dim3(ws::kThreads), S::SMEM, a);
}

template <typename TX, int BN>
void wgrad_tc_launch(ga3c_ctx* c, int li, const WgradArgs& a, dim3 grid, int tag = GA3C_K_WGRAD) {
  // ring cap by occupancy (DNN A: deep 0.85M, cap 3 0.95M, cap 2 / default
  // 1.01M samples/s -- occupancy beats depth)
  const int cap = ring_cap(c, (std::min(a.kc, a.npix) + 31) / 32, static_cast<long long>(grid.x) * grid.y * grid.z);
#define GA3C_F(C) wgrad_tc_launch_v<TX, BN, C>(c, li, a, grid, tag)
  GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
}

// u8 first conv layer with 32-byte window rows (k * Cin == 32): per-image
// pixel ranges staged whole by bulk copy (tc_wgrad_band.cuh) instead of
// im2col gathers; returns false when the shape does not qualify.
constexpr int kBandSmemMax = 220 * 1024;  // + the kernel's static shared memory <= 227 KB
bool layer_wgrad_band(ga3c_ctx* c, int li, const Layer& L, const uint8_t* x_in, const float* dout, int B,
                      long long in_stride, const GradMap& gm, float* part) {
  if (!L.is_conv || L.k * L.cin != 32 || L.k > 8 || L.out > wb::BN || L.out % 4 != 0 || L.in != 32 * L.k ||
      L.w_off % 4 != 0)
    return false;
  const long long bstride = in_stride > 0 ? in_stride : static_cast<long long>(L.ih) * L.iw * L.cin;
  const int rowb = L.iw * L.cin;
  if (rowb % 16 != 0 || bstride % 16 != 0 || reinterpret_cast<uintptr_t>(x_in) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(dout) % 16 != 0)
    return false;
  const int P = L.pixels(), nch = (P + 31) / 32;
  // CTAs per image: as the im2col path's split target (2x the SMs for a
  // context with the whole GPU, half its budget beside other trainers),
  // rounded down -- DNN A in the step, CTAs 40 / 80 / 120 / 240: 1.26M /
  // 1.25M / 1.23M / 1.19M samples/s, im2col path 1.21M; large s1 is
  // insensitive (148..1200: 105-107K)
  const bool whole = split_sms(c) >= kNumSMs;
  const int target = whole ? 2 * split_sms(c) : split_sms(c) / 2;
  int cpi = std::max(1, std::min(nch, target / B));
  const int cpc = (nch + cpi - 1) / cpi;
  cpi = (nch + cpc - 1) / cpc;
  int xband = 0, dband = 0;
  for (int j = 0; j < cpi; ++j) {
    const int p0 = 32 * j * cpc, p1 = std::min(P, 32 * (j + 1) * cpc);
    if (p0 >= p1) continue;
    const int y0 = (p0 / L.ow) * L.stride, y1 = ((p1 - 1) / L.ow) * L.stride + L.k;
    xband = std::max(xband, (y1 - y0) * rowb);
    dband = std::max(dband, (p1 - p0) * L.out * 4);
  }
  const int mt = (L.k + 3) / 4;
  const int smem = wb::smem_bytes(mt, xband, dband);
  const int splits = B * cpi;
  if (smem > kBandSmemMax || static_cast<std::size_t>(splits) * L.out * (L.in + 1) > kRegionFloats) return false;
  wb::BandArgs a{x_in, bstride, L.iw, L.cin, L.k, L.stride, L.ow, P, dout, L.out, L.out, L.in,
                 cpi, cpc, xband, dband, splits, part, gm, splits == 1};
  {
    Launch l(c, GA3C_K_WGRAD, li);
    if (mt == 1) {
      GA3C_SMEM_ONCE(wb::tc_wgrad_band_kernel<1>, kBandSmemMax);
      pdl_launch(c->cur, wb::tc_wgrad_band_kernel<1>, dim3(cpi, B), dim3(wb::kThreads), smem, a);
    } else {
      GA3C_SMEM_ONCE(wb::tc_wgrad_band_kernel<2>, kBandSmemMax);
      pdl_launch(c->cur, wb::tc_wgrad_band_kernel<2>, dim3(cpi, B), dim3(wb::kThreads), smem, a);
    }
  }
  if (splits > 1) {
    const std::size_t n = static_cast<std::size_t>(L.out) * (L.in + 1);
    Launch l(c, GA3C_K_SPLITK, li);
    if (splits > 16)
      pdl_launch(c->cur, splitk_wgrad8_kernel, dim3((unsigned)((n + 31) / 32)), dim3(256), 0, part, splits, L.out,
                 L.in, gm);
    else
      pdl_launch(c->cur, splitk_wgrad_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, part, splits, L.out,
                 L.in, gm);
  }
  return true;
}

// Tensor-core weight gradient; returns false when the shape needs the SIMT path.
template <typename TX>
bool layer_wgrad_tc(ga3c_ctx* c, int li, const Layer& L, const void* x_in, const float* dout, int B,
                    long long in_stride, const GradMap& gm, float* part) {
  if constexpr (sizeof(TX) == 1) {
    if (layer_wgrad_band(c, li, L, static_cast<const uint8_t*>(x_in), dout, B, in_stride, gm, part))
      return true;
  }
  const int npix = B * L.pixels();
  Seg X = L.is_conv ? conv_seg<TX>(L, x_in, in_stride)
                    : dense_seg(x_in, B, in_stride > 0 ? in_stride : L.in, L.in, sizeof(TX) == 1);
  X.rows = npix;
  if (!seg_ok(X, npix) || L.in % 32 != 0 || L.out % 4 != 0 || L.w_off % 4 != 0 ||
      (reinterpret_cast<uintptr_t>(dout) % 16) != 0)
    return false;
  const int mtiles = (L.in + 127) / 128;
  const int chunks = (npix + 31) / 32;
  // Narrowest N tile that still covers the outputs in one wave when the
  // reduction is too short to split (FC at trainer batch sizes): more CTAs,
  // each with a smaller epilogue.  When no tile fits one wave (large s1 FC,
  // 145 row tiles), the narrowest: small CTAs at ring cap 2 interleave with
  // the other trainers' kernels (large s1 105.5K -> 106.6K samples/s with
  // 32 vs 128, although the kernel alone is 24 vs 22 us).
  int bn = L.out <= 32 ? 32 : (L.out <= 64 ? 64 : 128);
  if (chunks < 4) {
    int pick = 32;
    for (int cand = 32; cand < bn; cand *= 2)
      if (mtiles * ((L.out + cand - 1) / cand) <= split_sms(c)) {
        pick = cand;
        break;
      }
    bn = std::min(bn, pick);
  }
  const int ntiles = (L.out + bn - 1) / bn;
  // A context with the whole GPU plans two CTAs per SM (ring cap 1), so the
  // conversion-heavy producers of one CTA overlap the other's; a context
  // sharing the GPU (a trainer beside other trainers) plans for a fraction
  // of its budget: fewer split partials to reduce on its critical path
  // (N_T = 3: x0.5 1.04M vs x1 1.00M, x2 0.96M samples/s; re-swept at N_T = 6,
  // two runs each: x0.1 1.389-1.393M, x0.15 1.390-1.392M, x0.2 1.386-1.387M,
  // x0.25 1.381-1.390M, x0.35 1.369-1.370M, x0.5 1.356-1.359M, x0.7 1.28-1.30M;
  // DNN A's conv2 weight gradient 26 -> 9 splits; large s1 whole-GPU x1 105K,
  // x0.5 94K).
  const bool whole = split_sms(c) >= kNumSMs;
  const double f = whole ? 2.0 : 0.15;
  const int wsms = std::max(1, static_cast<int>(f * split_sms(c)));
  int splits = std::max(1, std::min(chunks / 2, (wsms + mtiles * ntiles - 1) / (mtiles * ntiles)));
  while (splits > 1 && static_cast<std::size_t>(splits) * L.out * (L.in + 1) > kRegionFloats) --splits;
  const int kc = ((chunks + splits - 1) / splits) * 32;
  splits = (npix + kc - 1) / kc;
  WgradArgs a{X, dout, L.out, L.out, L.in, npix, kc, part, gm, splits == 1, 0, nullptr, nullptr, 0, 0};
  dim3 grid(mtiles, splits, ntiles);
  switch (bn) {
    case 32: wgrad_tc_launch<TX, 32>(c, li, a, grid); break;
    case 64: wgrad_tc_launch<TX, 64>(c, li, a, grid); break;
    default: wgrad_tc_launch<TX, 128>(c, li, a, grid); break;
  }
  if (splits > 1) {
    const std::size_t n = static_cast<std::size_t>(L.out) * (L.in + 1);
    Launch l(c, GA3C_K_SPLITK, li);
    if (splits > 16)
      pdl_launch(c->cur, splitk_wgrad8_kernel, dim3((unsigned)((n + 31) / 32)), dim3(256), 0, part,
                 splits, L.out, L.in, gm);
    else
      pdl_launch(c->cur, splitk_wgrad_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, part,
                 splits, L.out, L.in, gm);
  }
  return true;
}

template <typename T>
void layer_wgrad(ga3c_ctx* c, int li, const Layer& L, const void* x_in, const float* dout, int B,
                 long long in_stride) {
  GradMap gm{c->grad, c->flag, L.w_off, L.b_off, 0, 0, L.out, L.in};
  float* part = region(c, 1 + li);
  if (layer_wgrad_tc<T>(c, li, L, x_in, dout, B, in_stride, gm, part)) return;
  DenseT a{dout, L.out};  // (m = out channel, k = row) -> dout[row][m]
  if (L.is_conv) {
    WithOnes<Im2colB<T>> b;
    static_cast<Im2col<T>&>(b.l) = im2col_of<T>(L, x_in, in_stride);
    b.n_real = L.in;
    wgrad_gemm(c, li, a, b, gm, L.out, L.in + 1, B * L.pixels(), part);
  } else {
    WithOnes<DenseTIn<T>> b{
        DenseTIn<T>{static_cast<const T*>(x_in), in_stride > 0 ? static_cast<int>(in_stride) : L.in},
        L.in};
    wgrad_gemm(c, li, a, b, gm, L.out, L.in + 1, B, part);
  }
}

// FC input gradient on the tensor cores, computed transposed:
//   dX^T[i][b] = sum_o W[o][i] * dh^T[o][b]   (both operands MN-major)
// with the ReLU gate of the layer below fused into the store.  Needs the
// transposed output gradient the loss kernel writes for the top FC layer.
bool fc_dgrad_tc(ga3c_ctx* c, int li, const Layer& L, const float* theta, const float* doutT,
                 int ldT, const float* gate, float* din, int B) {
  Seg W = dense_seg(theta + L.w_off, L.out, L.in, L.in, false);
  W.rows = L.out;
  if (!seg_ok(W, L.out) || L.in % 32 != 0 || ldT % 4 != 0) return false;
  const int bn = B <= 32 ? 32 : (B <= 64 ? 64 : 128);  // batches above 128: grid.z = batch tiles
  // split the reduction over the layer's outputs across a cluster when the
  // row tiles alone cannot fill the SMs
  const int mtiles = (L.in + 127) / 128;
  const int chunks = (L.out + 31) / 32;
  int ks = std::max(1, std::min({8, chunks, cluster_sms(c) / mtiles}));
  const int kc = ((chunks + ks - 1) / ks) * 32;
  ks = (L.out + kc - 1) / kc;
  WgradArgs a{W, doutT, ldT, B, L.in, L.out, kc, nullptr, GradMap{}, 0, 1, din, gate, L.in, 0};
  dim3 grid(mtiles, ks, (B + bn - 1) / bn);
  switch (bn) {
    case 32: wgrad_tc_launch<float, 32>(c, li, a, grid, GA3C_K_DGRAD); break;
    case 64: wgrad_tc_launch<float, 64>(c, li, a, grid, GA3C_K_DGRAD); break;
    default: wgrad_tc_launch<float, 128>(c, li, a, grid, GA3C_K_DGRAD); break;
  }
  return true;
}

// Conv input gradient on the tensor cores (tc_dgrad.cuh): s*s stride-phase
// implicit GEMMs; false when the geometry needs the SIMT kernels.
template <int BN, int CAP>
void dgrad_tc_launch(ga3c_ctx* c, int li, const dg::DgradArgs& a, dim3 grid) {
  using S = dg::DgShape<BN, CAP>;
  auto kern = dg::tc_dgrad_kernel<BN, CAP>;
  GA3C_SMEM_ONCE(kern, S::SMEM);
  Launch l(c, GA3C_K_DGRAD, li);
  pdl_launch(c->cur, kern, grid, dim3(ws::kThreads), S::SMEM, a);
}

bool conv_dgrad_tc(ga3c_ctx* c, int li, const Layer& L, const float* theta, const float* dout,
                   const float* gate, float* din, int B) {
  if (L.k % L.stride != 0 || L.cout % 32 != 0 || L.cin % 16 != 0 || L.cin > 128) return false;
  const int T = L.k / L.stride;
  if (T * T * L.cout / 32 < 1) return false;
  dg::DgradArgs a{dout, theta + L.w_off, gate, din, B, L.ih, L.iw, L.cin, L.oh, L.ow, L.cout, L.k, L.stride, T};
  const int bn = L.cin <= 16 ? 16 : (L.cin <= 32 ? 32 : (L.cin <= 64 ? 64 : 128));
  const int a0 = (L.ih + L.stride - 1) / L.stride, b0 = (L.iw + L.stride - 1) / L.stride;
  const long long m0 = static_cast<long long>(B) * a0 * b0;
  const int ntiles = (L.cin + bn - 1) / bn;
  dim3 grid(static_cast<unsigned>((m0 + 127) / 128), L.stride * L.stride, ntiles);
  // ring cap by occupancy (large s1 conv2 dgrad: cap 0 = 97 us, 1 = 68 us,
  // 2 = 68 us, 3 = 97 us -- two CTAs per SM win)
  const int cap = ring_cap(c, T * T * L.cout / 32, static_cast<long long>(grid.x) * grid.y * grid.z);
  switch (bn) {
    case 16: {
#define GA3C_F(C) dgrad_tc_launch<16, C>(c, li, a, grid)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
    case 32: {
#define GA3C_F(C) dgrad_tc_launch<32, C>(c, li, a, grid)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
    case 64: {
#define GA3C_F(C) dgrad_tc_launch<64, C>(c, li, a, grid)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
    default: {
#define GA3C_F(C) dgrad_tc_launch<128, C>(c, li, a, grid)
      GA3C_CAP_SWITCH(cap, GA3C_F)
#undef GA3C_F
    } break;
  }
  return true;
}

void layer_dgrad(ga3c_ctx* c, int li, const Layer& L, const float* theta, const float* dout,
                 const float* gate, float* din, int B, const float* doutT = nullptr) {
  if (!L.is_conv && doutT && fc_dgrad_tc(c, li, L, theta, doutT, c->ldT, gate, din, B)) return;
  if (L.is_conv && conv_dgrad_tc(c, li, L, theta, dout, gate, din, B)) return;
  if (L.is_conv && L.cin % 16 == 0 && L.w_off % 4 == 0 && L.k == 4 && L.stride == 2 &&
      (L.cout == 32 || L.cout == 64)) {
    const int npix = B * L.ih * L.iw;
    const std::size_t smem = static_cast<std::size_t>(L.cout) * L.k * L.k * 16 * sizeof(float);
    auto kern = L.cout == 32 ? conv_dgrad_32x4s2_kernel : conv_dgrad_64x4s2_kernel;
    if (L.cout == 32) {
      GA3C_SMEM_ONCE(conv_dgrad_32x4s2_kernel, 200 * 1024);
    } else {
      GA3C_SMEM_ONCE(conv_dgrad_64x4s2_kernel, 200 * 1024);
    }
    Launch l(c, GA3C_K_DGRAD, li);
    pdl_launch(c->cur, kern, dim3((npix + 63) / 64, L.cin / 16), dim3(256), smem, dout, theta + L.w_off,
               gate, din, B, L.ih, L.iw, L.cin, L.oh, L.ow);
  } else if (L.is_conv && L.cin % 16 == 0 && L.cout % 4 == 0 && L.w_off % 4 == 0 &&
      static_cast<std::size_t>(L.cout) * L.k * L.k * 16 * sizeof(float) <= 200 * 1024) {
    const int npix = B * L.ih * L.iw;
    const std::size_t smem = static_cast<std::size_t>(L.cout) * L.k * L.k * 16 * sizeof(float);
    GA3C_SMEM_ONCE(conv_dgrad16_kernel, 200 * 1024);
    Launch l(c, GA3C_K_DGRAD, li);
    pdl_launch(c->cur, conv_dgrad16_kernel, dim3(dim3((npix + 63) / 64, L.cin / 16)), dim3(256), smem, 
        dout, theta + L.w_off, gate, din, B, L.ih, L.iw, L.cin, L.oh, L.ow, L.cout, L.k, L.stride);
  } else if (L.is_conv) {
    const std::size_t n = static_cast<std::size_t>(B) * L.ih * L.iw * L.cin;
    Launch l(c, GA3C_K_DGRAD, li);
    pdl_launch(c->cur, conv_dgrad_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, 
        dout, theta + L.w_off, gate, din, B, L.ih, L.iw, L.cin, L.oh, L.ow, L.cout, L.k, L.stride);
  } else {
    DenseK a{dout, L.out};
    DenseT w{theta + L.w_off, L.in};  // (n = i, k = o) -> W[o][i]
    launch_gemm(c, GA3C_K_DGRAD, li, a, w, EpiGate{din, gate, L.in}, B, L.in, L.out,
                plan_splits(c, B, L.in, L.out, false));
  }
}

// ------------------------------------------------------------- forward

__global__ void widen_u8_kernel(const uint8_t* __restrict__ x, float* __restrict__ y, std::size_t n) {
  pdl_enter();
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = static_cast<float>(x[i]) * (1.0f / 256.0f);
}

// What the heads consume: the last FC layer's split-K partials (+ its bias),
// or a finished h.
struct HeadsIn {
  const float* part = nullptr;
  int n_split = 0;
  const float* fc_bias = nullptr;
  float* h = nullptr;
};

// Trunk forward; then the predictor heads (softmax) unless `hin` is given,
// in which case the heads' inputs are returned for the trainer's fused
// heads + loss kernel.
int run_forward(ga3c_ctx* c, const float* theta, const void* d_in, bool u8, int B,
                long long in_stride = 0, HeadsIn* hin = nullptr) {
  const Layout& lo = c->m->lo;
  const void* x = d_in;
  bool x_u8 = u8;
  int n_split = 0;
  for (int li = 0; li < lo.n_trunk; ++li) {
    const Layer& L = lo.trunk[li];
    const bool last = li == lo.n_trunk - 1;
    if (L.is_conv) {
      if (x_u8)
        conv_forward<uint8_t>(c, li, L, theta, x, c->act[li], B, li == 0 ? in_stride : 0);
      else
        conv_forward<float>(c, li, L, theta, x, c->act[li], B, li == 0 ? in_stride : 0);
    } else {
      const long long st = li == 0 ? in_stride : 0;
      int s = x_u8 ? fc_forward<uint8_t>(c, li, L, theta, x, c->act[li], B, last, st)
                   : fc_forward<float>(c, li, L, theta, x, c->act[li], B, last, st);
      if (last) n_split = s;
    }
    x = c->act[li];
    x_u8 = false;
  }
  const int D = lo.head_in();
  const int A = lo.n_actions;
  const float* part = nullptr;
  const float* fc_bias = nullptr;
  float* h = nullptr;
  if (lo.n_trunk == 0) {
    if (u8) {
      // raw u8 input feeds the heads directly: widen once (k/256 is exact)
      const std::size_t n = static_cast<std::size_t>(B) * D;
      Launch l(c, GA3C_K_OTHER, -1);
      pdl_launch(c->cur, widen_u8_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, 
          static_cast<const uint8_t*>(d_in), c->hin, n);
      h = c->hin;
    } else {
      h = const_cast<float*>(static_cast<const float*>(d_in));
    }
  } else {
    h = c->act[lo.n_trunk - 1];
    if (!lo.trunk[lo.n_trunk - 1].is_conv && n_split > 0) {  // 0: the FC wrote h itself
      part = region(c, 0);
      fc_bias = theta + lo.trunk[lo.n_trunk - 1].b_off;
    }
  }
  if (hin) {
    hin->part = part;
    hin->n_split = n_split;
    hin->fc_bias = fc_bias;
    hin->h = h;
    return GA3C_OK;
  }
  const std::size_t smem = (static_cast<std::size_t>(D) * (A + 2) + 8 * (A + 1)) * sizeof(float);
  {
    Launch l(c, GA3C_K_HEADS, -1);
    pdl_launch(c->cur, heads_forward_kernel, dim3(B), dim3(256), smem, part, n_split, fc_bias, h, B, D, theta,
                                                      lo.policy.w_off, lo.policy.b_off, lo.value.w_off,
                                                      lo.value.b_off, A, c->pi32, c->pi64, c->v, c->v64);
  }
  return GA3C_OK;
}

int run_loss_grad(ga3c_ctx* c, const float* theta, const void* d_in, bool u8, const int32_t* d_act,
                  const double* d_rets, int B, bool apply_clip, long long in_stride = 0) {
  ga3c_model* m = c->m;
  const Layout& lo = m->lo;
  const int D = lo.head_in();
  const int A = lo.n_actions;
  HeadsIn hi;
  run_forward(c, theta, d_in, u8, B, in_stride, &hi);
  const float* h = hi.h;
  float* dh = lo.n_trunk ? c->dout[lo.n_trunk - 1] : nullptr;
  {
    const std::size_t smem = (static_cast<std::size_t>(D) * (A + 2) + 8 * (A + 1)) * sizeof(float);
    Launch l(c, GA3C_K_LOSS_BWD, -1);
    pdl_launch(c->cur, heads_loss_kernel, dim3(B), dim3(256), smem, hi.part, hi.n_split, hi.fc_bias, hi.h, B, D,
               theta, lo.policy.w_off, lo.policy.b_off, lo.value.w_off, lo.value.b_off, A, d_act, d_rets,
               m->hp.beta, m->hp.eps_log, m->hp.value_loss_weight, c->pi64, c->v, c->dhead, dh,
               lo.n_trunk ? c->dhT : nullptr, c->ldT, c->scal, c->flag);
  }
  // Backward DAG.  The critical path is the input-gradient chain
  // (loss -> dgrad L-1 -> ... -> dgrad 1 -> wgrad 0); the heads' and the
  // upper layers' weight gradients only need their layer's output gradient,
  // so they run on side streams as soon as it exists.  Every branch writes
  // disjoint dtheta ranges and its own split-K region, so the result is the
  // same bit for bit as the serial order.
  const bool heads_contig = lo.policy.b_off == lo.policy.w_off + static_cast<std::size_t>(A) * D &&
                            lo.value.w_off == lo.policy.b_off + A && lo.value.b_off == lo.value.w_off + D;
  bool used[2] = {true, false};
  fork_to(c, c->side[0]);
  if (heads_contig && A + 1 <= 32) {
    // heads weight gradient [A+1][D+1] = dhead^T [h | 1] + the loss sums
    const HeadsGrad hg{c->dhead, h, B, A, D, lo.policy.w_off, lo.policy.b_off, lo.value.w_off, lo.value.b_off,
                       c->scal, c->scal_sum};
    Launch l(c, GA3C_K_WGRAD, -1);
    pdl_launch(c->cur, heads_wgrad_kernel, dim3((D + 1 + 31) / 32), dim3(256), 0, hg, c->grad, c->flag);
  } else {
    // heads weight gradient: [A+1][D+1] = dhead^T [h | 1]
    GradMap gm{c->grad, c->flag, lo.policy.w_off, lo.policy.b_off, lo.value.w_off, lo.value.b_off, A, D};
    DenseT a{c->dhead, A + 1};
    WithOnes<DenseT> b{DenseT{h, D}, D};
    wgrad_gemm(c, -1, a, b, gm, A + 1, D + 1, B, region(c, kRegions - 1));
    Launch l(c, GA3C_K_OTHER, -1);
    pdl_launch(c->cur, scalars_kernel, dim3(1), dim3(32), 0, c->scal, B, c->scal_sum);
  }
  c->cur = c->stream;
  for (int li = lo.n_trunk - 1; li >= 0; --li) {
    const Layer& L = lo.trunk[li];
    const void* x_in = li == 0 ? d_in : c->act[li - 1];
    const bool in_u8 = li == 0 && u8;
    const long long st = li == 0 ? in_stride : 0;
    if (li > 0) {
      const int sd = li & 1;
      fork_to(c, c->side[sd]);
      used[sd] = true;
    }
    if (in_u8)
      layer_wgrad<uint8_t>(c, li, L, x_in, c->dout[li], B, st);
    else
      layer_wgrad<float>(c, li, L, x_in, c->dout[li], B, st);
    c->cur = c->stream;
    if (li > 0) {
      const float* doutT = li == lo.n_trunk - 1 ? c->dhT : nullptr;
      layer_dgrad(c, li, L, theta, c->dout[li], c->act[li - 1], c->dout[li - 1], B, doutT);
    }
  }
  for (int sd = 0; sd < 2; ++sd)
    if (used[sd]) join_from(c, c->side[sd]);
  if (apply_clip && m->hp.grad_clip_norm > 0.0) {
    {
      Launch l(c, GA3C_K_OTHER, -1);
      pdl_launch(c->cur, sumsq_kernel, dim3(kNumSMs), dim3(256), 0, c->grad, lo.total, c->clip_part);
    }
    Launch l(c, GA3C_K_OTHER, -1);
    pdl_launch(c->cur, clip_scale_kernel, dim3(kNumSMs), dim3(256), 0, c->grad, lo.total, c->clip_part, kNumSMs,
                                                      m->hp.grad_clip_norm);
  }
  return GA3C_OK;
}


// Frame store kernels.  A stacked pixel is one u32 (4 frames, oldest in the
// low byte); pushing shifts the oldest out and the new frame in, or fills
// all four with the new frame at an episode start.
//   idx = [agent | source slot | destination slot | reset] x n
__global__ void frames_push_kernel(uint32_t* __restrict__ ring, std::size_t px, int H,
                                   const uint32_t* __restrict__ newf, const int32_t* __restrict__ idx, int n,
                                   uint32_t* __restrict__ dense) {
  pdl_enter();
  const int i = blockIdx.y;
  const std::size_t q = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // 4 pixels
  if (q * 4 >= px) return;
  const int a = idx[i], src = idx[n + i], dst = idx[2 * n + i];
  const bool rst = idx[3 * n + i] != 0;
  const uint32_t f4 = newf[(static_cast<std::size_t>(i) * px) / 4 + q];
  const std::size_t so = ((static_cast<std::size_t>(a) * H + src) * px) + 4 * q;
  const std::size_t d0 = ((static_cast<std::size_t>(a) * H + dst) * px) + 4 * q;
  const uint4 old = *reinterpret_cast<const uint4*>(ring + so);
  const uint32_t o[4] = {old.x, old.y, old.z, old.w};
  uint32_t r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t fb = (f4 >> (8 * j)) & 0xFFu;
    r[j] = rst ? fb * 0x01010101u : (o[j] >> 8) | (fb << 24);
  }
  const uint4 w = make_uint4(r[0], r[1], r[2], r[3]);
  *reinterpret_cast<uint4*>(ring + d0) = w;
  if (dense) *reinterpret_cast<uint4*>(dense + static_cast<std::size_t>(i) * px + 4 * q) = w;
}

//   idx = [agent | slot] x B  ->  dense [B][state]
__global__ void frames_gather_kernel(const uint32_t* __restrict__ ring, std::size_t px, int H,
                                     const int32_t* __restrict__ idx, int B, uint32_t* __restrict__ out) {
  pdl_enter();
  const int b = blockIdx.y;
  const std::size_t q = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q * 4 >= px) return;
  const std::size_t so = ((static_cast<std::size_t>(idx[b]) * H + idx[B + b]) * px) + 4 * q;
  *reinterpret_cast<uint4*>(out + static_cast<std::size_t>(b) * px + 4 * q) =
      *reinterpret_cast<const uint4*>(ring + so);
}


// RMSProp from slot `src` into slot `dst` with the gradient (and its
// non-finite flag) of context `g` (default: c itself), on c's stream.
void launch_rmsprop(ga3c_ctx* c, const Slot& src, const Slot& dst, unsigned long long* ver,
                    const ga3c_ctx* g = nullptr) {
  if (!g) g = c;
  const ga3c_hyper& hp = c->m->hp;
  const std::size_t n = c->m->lo.total;
  const float alpha = static_cast<float>(hp.alpha);
  const float oma = static_cast<float>(1.0 - hp.alpha);
  const std::size_t n4 = (n + 3) / 4;
  // the gradient's context sharing the GPU (a trainer beside others): 2
  // CTAs per SM, else 8 (DNN A at N_T = 6, two runs each: 74 -> 1.401M,
  // 148 -> 1.456-1.464M, 296 -> 1.481-1.483M, 663 = one float4 per thread
  // -> 1.473-1.478M samples/s); elementwise, so bitwise either way
  const int cap = split_sms(g) < kNumSMs ? 2 * kNumSMs : 8 * kNumSMs;
  unsigned blocks = (unsigned)std::min<std::size_t>((n4 + 255) / 256, cap);
  if (blocks == 0) blocks = 1;
  Launch l(c, GA3C_K_RMSPROP, -1);
  pdl_launch(c->cur, rmsprop_kernel, dim3(blocks), dim3(256), 0, src.theta, src.g, (const float*)g->grad, dst.theta,
             dst.g, n, (const int*)g->flag, ver, alpha, oma, static_cast<float>(hp.eta),
                                                static_cast<float>(hp.eps_rms));
}

int set_device(ga3c_model* m) {
  if (cudaSetDevice(m->device) != cudaSuccess) return GA3C_CUDA_ERROR;
  return GA3C_OK;
}

// The apply-in-flight state of slot s, read under read_m.
cudaEvent_t pending_event(ga3c_model* m, int s) {
  std::lock_guard<std::mutex> lk(m->read_m);
  const Slot& sl = m->slots[s];
  return sl.pending ? sl.ready : nullptr;
}

// Orders c's stream after an asynchronous apply still writing slot s.
void wait_slot(ga3c_ctx* c, int s) {
  if (c->capturing) return;
  if (cudaEvent_t e = pending_event(c->m, s)) cudaStreamWaitEvent(c->stream, e, 0);
}

// Host side: waits until slot s is written.
void sync_slot(ga3c_model* m, int s) {
  if (cudaEvent_t e = pending_event(m, s)) cudaEventSynchronize(e);
}

// Allocates (or reuses) a slot with no readers that is not the current one.
// Caller holds update_m and read_m.
int free_slot_locked(ga3c_model* m) {
  for (int i = 0; i < (int)m->slots.size(); ++i)
    if (i != m->cur && m->slots[i].refs == 0) return i;
  Slot s;
  const std::size_t bytes = m->lo.total * sizeof(float);
  if (cudaMalloc(&s.theta, bytes) != cudaSuccess) return -1;
  if (cudaMalloc(&s.g, bytes) != cudaSuccess) {
    cudaFree(s.theta);
    return -1;
  }
  if (!m->slots.push_back(s)) {
    cudaFree(s.theta);
    cudaFree(s.g);
    return -1;
  }
  return (int)m->slots.size() - 1;
}

bool all_finite(const float* x, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

}  // namespace

// =================================================================== C ABI

extern "C" {

const char* ga3c_status_string(int s) {
  switch (s) {
    case GA3C_OK: return "ok";
    case GA3C_INVALID_ARGUMENT: return "invalid argument";
    case GA3C_NONFINITE_INPUT: return "non-finite input";
    case GA3C_CUDA_ERROR: return "cuda error";
    case GA3C_NCCL_ERROR: return "nccl error";
    case GA3C_NOT_APPLIED: return "update not applied (non-finite gradient)";
    case GA3C_OUT_OF_MEMORY: return "out of memory";
    default: return "unknown status";
  }
}


void ga3c_default_hyper(ga3c_hyper* hp) {
  hp->gamma = 0.99;
  hp->t_max = 5;
  hp->beta = 0.01;
  hp->eps_log = 1e-6;
  hp->eta = 3e-4;
  hp->alpha = 0.99;
  hp->eps_rms = 1e-8;
  hp->value_loss_weight = 0.5;
  hp->grad_clip_norm = 0.0;
  hp->clip_rewards = 0;
}

int ga3c_validate_spec(const ga3c_net_spec* s) {
  if (!s) return GA3C_INVALID_ARGUMENT;
  return validate_spec(*s);
}

int ga3c_validate_hyper(const ga3c_hyper* hp) {
  if (!hp) return GA3C_INVALID_ARGUMENT;
  return validate_hyper(*hp);
}

size_t ga3c_param_count(const ga3c_net_spec* s) {
  if (!s || validate_spec(*s) != GA3C_OK) return 0;
  return layout_of(*s).total;
}

size_t ga3c_input_dim(const ga3c_net_spec* s) {
  if (!s) return 0;
  return static_cast<size_t>(s->in_h) * s->in_w * s->in_c;
}

int ga3c_init_params(const ga3c_net_spec* s, uint64_t seed, double* theta64, float* theta32) {
  if (!s || validate_spec(*s) != GA3C_OK) return GA3C_INVALID_ARGUMENT;
  const Layout lo = layout_of(*s);
  std::vector<double> t(lo.total);
  init_params(lo, seed, t.data());
  if (theta64) std::memcpy(theta64, t.data(), lo.total * sizeof(double));
  if (theta32)
    for (std::size_t i = 0; i < lo.total; ++i) theta32[i] = static_cast<float>(t[i]);
  return GA3C_OK;
}

ga3c_model* ga3c_model_create(const ga3c_net_spec* spec, const ga3c_hyper* hp, int device,
                              int* status) {
  auto fail = [&](int st, const char* msg) -> ga3c_model* {
    g_tls_error = msg;
    if (status) *status = st;
    return nullptr;
  };
  if (!spec || !hp) return fail(GA3C_INVALID_ARGUMENT, "null spec/hyper");
  if (validate_spec(*spec) != GA3C_OK) return fail(GA3C_INVALID_ARGUMENT, "invalid NetworkSpec");
  if (validate_hyper(*hp) != GA3C_OK) return fail(GA3C_INVALID_ARGUMENT, "invalid Hyperparams");
  if (spec->n_actions > kMaxActions) return fail(GA3C_INVALID_ARGUMENT, "n_actions > 64 unsupported");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(GA3C_CUDA_ERROR, "no CUDA device (this library has no CPU path)");
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
    return fail(GA3C_CUDA_ERROR, "device is not sm_100 (B200)");
  if (cudaSetDevice(device) != cudaSuccess) return fail(GA3C_CUDA_ERROR, "cudaSetDevice failed");
  auto* m = new ga3c_model();
  m->spec = *spec;
  m->hp = *hp;
  m->lo = layout_of(*spec);
  m->device = device;
  if ((static_cast<std::size_t>(m->lo.head_in()) * (spec->n_actions + 2) + 8 * (spec->n_actions + 1)) *
          sizeof(float) > 200 * 1024) {
    delete m;
    return fail(GA3C_INVALID_ARGUMENT, "head input too wide: the heads' weights must fit shared memory");
  }
  Slot s;
  const std::size_t bytes = m->lo.total * sizeof(float);
  if (cudaMalloc(&s.theta, bytes) != cudaSuccess || cudaMalloc(&s.g, bytes) != cudaSuccess ||
      cudaMemset(s.theta, 0, bytes) != cudaSuccess || cudaMemset(s.g, 0, bytes) != cudaSuccess) {
    delete m;
    return fail(GA3C_OUT_OF_MEMORY, "parameter allocation failed");
  }
  m->slots.push_back(s);
  m->cur = 0;
  if (status) *status = GA3C_OK;
  return m;
}

void ga3c_model_destroy(ga3c_model* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  cudaDeviceSynchronize();  // asynchronous applies may still be writing slots
  for (auto& s : m->slots) {
    cudaFree(s.theta);
    cudaFree(s.g);
    if (s.ready) cudaEventDestroy(s.ready);
  }
  if (m->apply_done) cudaEventDestroy(m->apply_done);
  delete m;
}

int ga3c_model_load(ga3c_model* m, const float* theta, const float* g, uint64_t version) {
  if (!m || !theta) return GA3C_INVALID_ARGUMENT;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  std::lock_guard<std::mutex> ulk(m->update_m);
  if (m->apply_pending) GA3C_CUDA(cudaEventSynchronize(m->apply_done));  // no write in flight
  int f;
  {
    std::lock_guard<std::mutex> lk(m->read_m);
    f = free_slot_locked(m);
  }
  if (f < 0) return GA3C_OUT_OF_MEMORY;
  const std::size_t bytes = m->lo.total * sizeof(float);
  GA3C_CUDA(cudaMemcpy(m->slots[f].theta, theta, bytes, cudaMemcpyHostToDevice));
  if (g)
    GA3C_CUDA(cudaMemcpy(m->slots[f].g, g, bytes, cudaMemcpyHostToDevice));
  else
    GA3C_CUDA(cudaMemset(m->slots[f].g, 0, bytes));
  std::lock_guard<std::mutex> lk(m->read_m);
  m->slots[f].version = version;
  m->cur = f;
  return GA3C_OK;
}

int ga3c_model_read(ga3c_model* m, float* theta, float* g, uint64_t* version) {
  if (!m) return GA3C_INVALID_ARGUMENT;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  int s;
  uint64_t v;
  if (ga3c_snapshot_acquire(m, &s, &v)) return GA3C_INVALID_ARGUMENT;
  sync_slot(m, s);
  const std::size_t bytes = m->lo.total * sizeof(float);
  int rc = GA3C_OK;
  if (theta && cudaMemcpy(theta, m->slots[s].theta, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = GA3C_CUDA_ERROR;
  if (g && cudaMemcpy(g, m->slots[s].g, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = GA3C_CUDA_ERROR;
  if (version) *version = v;
  ga3c_snapshot_release(m, s);
  if (rc) set_err("ga3c_model_read: copy failed");
  return rc;
}

int ga3c_model_read_slot(ga3c_model* m, int slot, float* theta, float* g) {
  if (!m || slot < 0 || slot >= m->slots.size()) return GA3C_INVALID_ARGUMENT;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  GA3C_CUDA(cudaDeviceSynchronize());
  const std::size_t bytes = m->lo.total * sizeof(float);
  if (theta) GA3C_CUDA(cudaMemcpy(theta, m->slots[slot].theta, bytes, cudaMemcpyDeviceToHost));
  if (g) GA3C_CUDA(cudaMemcpy(g, m->slots[slot].g, bytes, cudaMemcpyDeviceToHost));
  return GA3C_OK;
}

uint64_t ga3c_model_version(ga3c_model* m) {
  std::lock_guard<std::mutex> lk(m->read_m);
  return m->slots[m->cur].version;
}

size_t ga3c_model_param_count(ga3c_model* m) { return m ? m->lo.total : 0; }

int ga3c_model_n_actions(ga3c_model* m) { return m ? m->lo.n_actions : 0; }

int ga3c_snapshot_acquire(ga3c_model* m, int* slot, uint64_t* version) {
  if (!m || !slot) return GA3C_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(m->read_m);
  *slot = m->cur;
  m->slots[m->cur].refs++;
  if (version) *version = m->slots[m->cur].version;
  return GA3C_OK;
}

int ga3c_snapshot_release(ga3c_model* m, int slot) {
  if (!m) return GA3C_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(m->read_m);
  if (slot < 0 || slot >= (int)m->slots.size() || m->slots[slot].refs <= 0)
    return GA3C_INVALID_ARGUMENT;
  m->slots[slot].refs--;
  return GA3C_OK;
}

const char* ga3c_model_last_error(ga3c_model* m) {
  if (!m) return g_tls_error.c_str();
  std::lock_guard<std::mutex> lk(m->err_m);
  return m->last_error.empty() ? g_tls_error.c_str() : m->last_error.c_str();
}

ga3c_ctx* ga3c_ctx_create(ga3c_model* m, int max_batch, int* status) {
  if (!m || max_batch < 1) {
    if (status) *status = GA3C_INVALID_ARGUMENT;
    return nullptr;
  }
  if (set_device(m)) {
    if (status) *status = GA3C_CUDA_ERROR;
    return nullptr;
  }
  auto* c = new ga3c_ctx();
  c->m = m;
  c->max_batch = max_batch;
  const Layout& lo = m->lo;
  const std::size_t B = max_batch;
  // The context stream carries the critical path (forward, loss, the
  // input-gradient chain, RMSProp) at the highest priority; the side
  // streams of the backward DAG (weight gradients) fill the SMs it leaves.
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  bool ok = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) == cudaSuccess;
  c->cur = c->stream;
  for (auto& sd : c->side)
    if (ok) ok = cudaStreamCreateWithPriority(&sd, cudaStreamNonBlocking, prio_lo) == cudaSuccess;
  for (auto& e : c->evs)
    if (ok) ok = cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  auto alloc = [&](auto** p, std::size_t bytes) {
    if (!ok) return;
    ok = cudaMalloc(reinterpret_cast<void**>(p), std::max<std::size_t>(bytes, 16)) == cudaSuccess;
  };
  alloc(&c->d_in, B * lo.in_dim * sizeof(float));
  for (int i = 0; i < lo.n_trunk; ++i) alloc(&c->act[i], B * lo.trunk[i].out_dim() * sizeof(float));
  for (int i = 0; i < lo.n_trunk; ++i) alloc(&c->dout[i], B * lo.trunk[i].out_dim() * sizeof(float));
  if (lo.n_trunk == 0) alloc(&c->hin, B * lo.in_dim * sizeof(float));
  alloc(&c->pi32, B * lo.n_actions * sizeof(float));
  alloc(&c->pi64, B * lo.n_actions * sizeof(double));
  alloc(&c->v, B * sizeof(float));
  alloc(&c->v64, B * sizeof(double));
  alloc(&c->dhead, B * (lo.n_actions + 1) * sizeof(float));
  c->ldT = static_cast<int>((B + 3) / 4 * 4);
  alloc(&c->dhT, static_cast<std::size_t>(lo.head_in()) * c->ldT * sizeof(float));
  if (ok) ok = cudaMemset(c->dhT, 0, static_cast<std::size_t>(lo.head_in()) * c->ldT * sizeof(float)) == cudaSuccess;
  alloc(&c->scal, B * 3 * sizeof(double));
  alloc(&c->scal_sum, 3 * sizeof(double));
  alloc(&c->d_actions, B * sizeof(int32_t));
  alloc(&c->d_rets, B * sizeof(double));
  alloc(&c->grad, lo.total * sizeof(float));
  alloc(&c->flag, sizeof(int));
  alloc(&c->dev_version, sizeof(unsigned long long));
  alloc(&c->part, kPartFloats * sizeof(float));
  alloc(&c->clip_part, kNumSMs * sizeof(double));
  if (ok) ok = cudaMallocHost(&c->h_flag, sizeof(int)) == cudaSuccess;
  c->stage_bytes = std::max<std::size_t>(kStageBytes, static_cast<std::size_t>(B) * 64);
  if (ok) ok = cudaMallocHost(&c->h_stage, c->stage_bytes) == cudaSuccess;
  alloc(&c->d_stage, c->stage_bytes);
  if (ok) ok = cudaMemset(c->dev_version, 0, sizeof(unsigned long long)) == cudaSuccess;
  if (ok) ok = cudaMemset(c->flag, 0, sizeof(int)) == cudaSuccess;
  if (ok) {
    const int max_smem = 200 * 1024;
    ok = cudaFuncSetAttribute(heads_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              max_smem) == cudaSuccess &&
         cudaFuncSetAttribute(heads_loss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem) ==
             cudaSuccess;
  }
  if (!ok) {
    g_tls_error = "ga3c_ctx_create: device allocation failed";
    ga3c_ctx_destroy(c);
    if (status) *status = GA3C_OUT_OF_MEMORY;
    return nullptr;
  }
  if (status) *status = GA3C_OK;
  return c;
}

void ga3c_ctx_destroy(ga3c_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->m->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  void* ps[] = {c->d_in, c->hin, c->pi32, c->pi64, c->v, c->v64, c->dhead, c->dhT, c->scal,
                c->scal_sum, c->d_actions, c->d_rets, c->grad, c->flag, c->dev_version, c->part,
                c->clip_part, c->r_rew, c->r_off, c->r_term, c->r_boot, c->r_out, c->f_idx, c->d_stage};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (auto* a : c->act)
    if (a) cudaFree(a);
  for (auto* a : c->dout)
    if (a) cudaFree(a);
  for (auto sd : c->side)
    if (sd) {
      cudaStreamSynchronize(sd);
      cudaStreamDestroy(sd);
    }
  for (auto e : c->evs)
    if (e) cudaEventDestroy(e);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->pend.active) {
    cudaEventSynchronize(c->pend.ev);
    if (c->pend.pinned) ga3c_snapshot_release(c->m, c->pend.slot);
  }
  if (c->pend.ev) cudaEventDestroy(c->pend.ev);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto e : c->events) cudaEventDestroy(e);
  for (auto g : c->graphs) cudaGraphExecDestroy(g);
  for (auto& kv : c->tf_graphs) cudaGraphExecDestroy(kv.second);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void* ga3c_ctx_stream(ga3c_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int ga3c_ctx_sync(ga3c_ctx* c) {
  if (!c) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  GA3C_CUDA(cudaStreamSynchronize(c->stream));
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

uint64_t ga3c_ctx_launches(ga3c_ctx* c) { return c ? c->launches : 0; }

static bool stride_ok(const ga3c_model* m, long long stride) {
  if (stride == 0) return true;
  if (stride < m->lo.in_dim) return false;
  return m->lo.n_trunk > 0 || stride == m->lo.in_dim;
}

int ga3c_forward_dev(ga3c_ctx* c, int slot, const void* d_states, int states_are_u8,
                     long long state_stride, int B, float* d_pi, float* d_v) {
  if (!c || B < 0 || B > c->max_batch || slot < 0 || slot >= (int)c->m->slots.size() ||
      !stride_ok(c->m, state_stride))
    return GA3C_INVALID_ARGUMENT;
  if (B == 0) return GA3C_OK;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  const float* theta = m->slots[slot].theta;
  wait_slot(c, slot);
  run_forward(c, theta, d_states, states_are_u8 != 0, B, state_stride);
  const int A = m->lo.n_actions;
  if (d_pi && d_pi != c->pi32)
    GA3C_CUDA(cudaMemcpyAsync(d_pi, c->pi32, sizeof(float) * B * A, cudaMemcpyDeviceToDevice, c->stream));
  if (d_v && d_v != c->v)
    GA3C_CUDA(cudaMemcpyAsync(d_v, c->v, sizeof(float) * B, cudaMemcpyDeviceToDevice, c->stream));
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

// pi/v receive fp32 copies, pi64/v64 the fp64 softmax and widened V (either
// pair may be null, not both).
static int forward_host(ga3c_ctx* c, int slot, const void* states, bool u8, int B, float* pi,
                        float* v, uint64_t* version_used, double* pi64 = nullptr, double* v64 = nullptr) {
  if (!c || B < 0 || B > c->max_batch || (B > 0 && (!states || (!(pi && v) && !(pi64 && v64)))))
    return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  const std::size_t dim = m->lo.in_dim;
  if (!u8 && !all_finite(static_cast<const float*>(states), dim * B)) return GA3C_NONFINITE_INPUT;
  if (set_device(m)) return GA3C_CUDA_ERROR;
  int s = slot;
  uint64_t ver = 0;
  const bool pinned_here = slot < 0;
  if (pinned_here) {
    ga3c_snapshot_acquire(m, &s, &ver);
  } else {
    if (slot >= (int)m->slots.size()) return GA3C_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(m->read_m);
    ver = m->slots[slot].version;
  }
  int rc = GA3C_OK;
  if (B > 0) {
    const std::size_t bytes = dim * B * (u8 ? 1 : sizeof(float));
    if (cudaMemcpyAsync(c->d_in, states, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      rc = GA3C_CUDA_ERROR;
    if (!rc) {
      wait_slot(c, s);
      run_forward(c, m->slots[s].theta, c->d_in, u8, B);
    }
    const int A = m->lo.n_actions;
    if (!rc && pi && cudaMemcpyAsync(pi, c->pi32, sizeof(float) * B * A, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      rc = GA3C_CUDA_ERROR;
    if (!rc && v && cudaMemcpyAsync(v, c->v, sizeof(float) * B, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      rc = GA3C_CUDA_ERROR;
    if (!rc && pi64 &&
        cudaMemcpyAsync(pi64, c->pi64, sizeof(double) * B * A, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      rc = GA3C_CUDA_ERROR;
    if (!rc && v64 && cudaMemcpyAsync(v64, c->v64, sizeof(double) * B, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      rc = GA3C_CUDA_ERROR;
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      rc = GA3C_CUDA_ERROR;
      set_err(std::string("forward: ") + cudaGetErrorString(e));
    }
  }
  if (pinned_here) ga3c_snapshot_release(m, s);
  if (version_used) *version_used = ver;
  return rc;
}

int ga3c_forward_u8(ga3c_ctx* c, int slot, const uint8_t* frames, int B, float* pi, float* v,
                    uint64_t* version_used) {
  return forward_host(c, slot, frames, true, B, pi, v, version_used);
}

int ga3c_forward_f32(ga3c_ctx* c, int slot, const float* states, int B, float* pi, float* v,
                     uint64_t* version_used) {
  return forward_host(c, slot, states, false, B, pi, v, version_used);
}

int ga3c_forward64_u8(ga3c_ctx* c, int slot, const uint8_t* frames, int B, double* pi, double* v,
                      uint64_t* version_used) {
  return forward_host(c, slot, frames, true, B, nullptr, nullptr, version_used, pi, v);
}

int ga3c_forward64_f32(ga3c_ctx* c, int slot, const float* states, int B, double* pi, double* v,
                       uint64_t* version_used) {
  return forward_host(c, slot, states, false, B, nullptr, nullptr, version_used, pi, v);
}

int ga3c_loss_grad_dev(ga3c_ctx* c, int slot, const void* d_states, int states_are_u8,
                       long long state_stride, const int32_t* d_actions, const double* d_returns,
                       int B, int apply_clip) {
  if (!c || B < 1 || B > c->max_batch || slot < 0 || slot >= (int)c->m->slots.size() ||
      !stride_ok(c->m, state_stride))
    return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  wait_slot(c, slot);
  c->grad_flag = -1;
  run_loss_grad(c, m->slots[slot].theta, d_states, states_are_u8 != 0, d_actions, d_returns, B,
                apply_clip != 0, state_stride);
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

static int loss_grad_host(ga3c_ctx* c, int slot, const void* states, bool u8,
                          const int32_t* actions, const double* rets, int B, int apply_clip,
                          float* dtheta, double* scalars) {
  if (!c || B < 1 || B > c->max_batch || !states || !actions || !rets) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  const std::size_t dim = m->lo.in_dim;
  for (int b = 0; b < B; ++b) {
    if (!std::isfinite(rets[b])) return GA3C_NONFINITE_INPUT;
    if (actions[b] < 0 || actions[b] >= m->lo.n_actions) return GA3C_INVALID_ARGUMENT;
  }
  if (!u8 && !all_finite(static_cast<const float*>(states), dim * B)) return GA3C_NONFINITE_INPUT;
  if (set_device(m)) return GA3C_CUDA_ERROR;
  int s = slot;
  const bool pinned_here = slot < 0;
  if (pinned_here) ga3c_snapshot_acquire(m, &s, nullptr);
  int rc = GA3C_OK;
  const std::size_t bytes = dim * B * (u8 ? 1 : sizeof(float));
  if (cudaMemcpyAsync(c->d_in, states, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(c->d_actions, actions, sizeof(int32_t) * B, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(c->d_rets, rets, sizeof(double) * B, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    rc = GA3C_CUDA_ERROR;
  c->grad_flag = -1;
  if (!rc) {
    wait_slot(c, s);
    run_loss_grad(c, m->slots[s].theta, c->d_in, u8, c->d_actions, c->d_rets, B, apply_clip != 0);
  }
  if (!rc && cudaMemcpyAsync(c->h_flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    rc = GA3C_CUDA_ERROR;
  if (!rc && dtheta &&
      cudaMemcpyAsync(dtheta, c->grad, sizeof(float) * m->lo.total, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    rc = GA3C_CUDA_ERROR;
  if (!rc && scalars &&
      cudaMemcpyAsync(scalars, c->scal_sum, sizeof(double) * 3, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    rc = GA3C_CUDA_ERROR;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    rc = GA3C_CUDA_ERROR;
    set_err(std::string("loss_grad: ") + cudaGetErrorString(e));
  }
  if (!rc) c->grad_flag = *c->h_flag;
  if (pinned_here) ga3c_snapshot_release(m, s);
  return rc;
}

int ga3c_loss_grad_u8(ga3c_ctx* c, int slot, const uint8_t* frames, const int32_t* actions,
                      const double* returns, int B, int apply_clip, float* dtheta, double* scalars) {
  return loss_grad_host(c, slot, frames, true, actions, returns, B, apply_clip, dtheta, scalars);
}

int ga3c_loss_grad_f32(ga3c_ctx* c, int slot, const float* states, const int32_t* actions,
                       const double* returns, int B, int apply_clip, float* dtheta, double* scalars) {
  return loss_grad_host(c, slot, states, false, actions, returns, B, apply_clip, dtheta, scalars);
}

float* ga3c_ctx_grad(ga3c_ctx* c) { return c ? c->grad : nullptr; }

ga3c_model* ga3c_ctx_model(ga3c_ctx* c) { return c ? c->m : nullptr; }

const double* ga3c_ctx_last_values(ga3c_ctx* c) { return c ? c->v64 : nullptr; }

int ga3c_ctx_read_grad(ga3c_ctx* c, float* dtheta, double* scalars) {
  if (!c) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (dtheta)
    GA3C_CUDA(cudaMemcpyAsync(dtheta, c->grad, sizeof(float) * m->lo.total, cudaMemcpyDeviceToHost, c->stream));
  if (scalars)
    GA3C_CUDA(cudaMemcpyAsync(scalars, c->scal_sum, sizeof(double) * 3, cudaMemcpyDeviceToHost, c->stream));
  GA3C_CUDA(cudaStreamSynchronize(c->stream));
  return GA3C_OK;
}

int ga3c_clip_grad(ga3c_ctx* c) {
  if (!c) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (m->hp.grad_clip_norm > 0.0) {
    {
      Launch l(c, GA3C_K_OTHER, -1);
      pdl_launch(c->cur, sumsq_kernel, dim3(kNumSMs), dim3(256), 0, c->grad, m->lo.total, c->clip_part);
    }
    Launch l(c, GA3C_K_OTHER, -1);
    pdl_launch(c->cur, clip_scale_kernel, dim3(kNumSMs), dim3(256), 0, c->grad, m->lo.total, c->clip_part, kNumSMs,
                                                      m->hp.grad_clip_norm);
  }
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

int ga3c_check_grad(ga3c_ctx* c, ga3c_ctx* grad_from) {
  if (!c || (grad_from && grad_from->m != c->m)) return GA3C_INVALID_ARGUMENT;
  ga3c_ctx* g = grad_from ? grad_from : c;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  GA3C_CUDA(cudaMemsetAsync(g->flag, 0, sizeof(int), c->cur));
  {
    Launch l(c, GA3C_K_OTHER, -1);
    pdl_launch(c->cur, check_finite_kernel, dim3(kNumSMs), dim3(256), 0, (const float*)g->grad, m->lo.total, g->flag);
  }
  g->grad_flag = -1;
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

int ga3c_rmsprop_flat(const ga3c_hyper* hp, int device, size_t n, float* theta, float* g, const float* dtheta,
                      int* applied) {
  if (!hp || !theta || !g || !dtheta || validate_hyper(*hp) != GA3C_OK) return GA3C_INVALID_ARGUMENT;
  if (applied) *applied = 0;
  if (n == 0) {
    if (applied) *applied = 1;
    return GA3C_OK;
  }
  auto set_err = [&](const std::string& e) { g_tls_error = e; };
  GA3C_CUDA(cudaSetDevice(device));
  float* d = nullptr;
  int* flag = nullptr;
  const std::size_t bytes = n * sizeof(float);
  // the kernel moves float4s: every sub-buffer starts 256-byte aligned
  const std::size_t np = (n + 63) / 64 * 64;
  GA3C_CUDA(cudaMalloc(&d, (3 * np + 64) * sizeof(float)));
  float* th = d;
  float* gg = d + np;
  float* dt = d + 2 * np;
  flag = reinterpret_cast<int*>(d + 3 * np);
  int h_flag = 1;
  cudaError_t e = cudaMemcpy(th, theta, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(gg, g, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dt, dtheta, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(flag, 0, sizeof(int));
  if (e == cudaSuccess) {
    check_finite_kernel<<<kNumSMs, 256>>>(dt, n, flag);
    const std::size_t n4 = (n + 3) / 4;
    const unsigned blocks = (unsigned)std::max<std::size_t>(1, std::min<std::size_t>((n4 + 255) / 256, 8 * kNumSMs));
    rmsprop_kernel<<<blocks, 256>>>(th, gg, dt, th, gg, n, flag, nullptr, static_cast<float>(hp->alpha),
                                    static_cast<float>(1.0 - hp->alpha), static_cast<float>(hp->eta),
                                    static_cast<float>(hp->eps_rms));
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && !h_flag) e = cudaMemcpy(theta, th, bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && !h_flag) e = cudaMemcpy(g, gg, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  GA3C_CUDA(e);
  if (h_flag) return GA3C_NOT_APPLIED;
  if (applied) *applied = 1;
  return GA3C_OK;
}

int ga3c_apply_rmsprop(ga3c_ctx* c, const float* dtheta, int* applied, uint64_t* applied_on) {
  if (!c) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  const std::size_t n = m->lo.total;
  // The gradient's non-finite flag is already on the host when this
  // context's last gradient came from a host-buffer call (which waited for
  // it): then the step is applied asynchronously -- RMSProp is enqueued on
  // this context's stream, the destination slot is published at once with
  // an event that every later reader of the slot (device or host) orders
  // after, and the call returns without a device round trip.
  const bool async = !dtheta && c->grad_flag >= 0 && !c->capturing;
  if (async && c->grad_flag) {  // rejected (nnet.cpp:299-301): nothing changes
    c->grad_flag = -1;
    if (applied) *applied = 0;
    return GA3C_NOT_APPLIED;
  }
  std::lock_guard<std::mutex> ulk(m->update_m);
  int src, dst;
  {
    std::lock_guard<std::mutex> lk(m->read_m);
    src = m->cur;
    m->slots[src].refs++;
    dst = free_slot_locked(m);
  }
  auto unpin = [&]() {
    std::lock_guard<std::mutex> lk(m->read_m);
    m->slots[src].refs--;
  };
  if (dst < 0) {
    unpin();
    return GA3C_OUT_OF_MEMORY;
  }
  // every write orders after the previous asynchronous apply (it read its
  // source and wrote its destination, either of which may be src / dst here)
  if (m->apply_pending) GA3C_CUDA(cudaStreamWaitEvent(c->stream, m->apply_done, 0));
  if (async) {
    c->grad_flag = -1;
    Slot& d = m->slots[dst];
    if (!d.ready) GA3C_CUDA(cudaEventCreateWithFlags(&d.ready, cudaEventDisableTiming));
    if (!m->apply_done) GA3C_CUDA(cudaEventCreateWithFlags(&m->apply_done, cudaEventDisableTiming));
    launch_rmsprop(c, m->slots[src], d, nullptr);
    GA3C_CUDA(cudaEventRecord(d.ready, c->stream));
    GA3C_CUDA(cudaEventRecord(m->apply_done, c->stream));
    {
      std::lock_guard<std::mutex> lk(m->read_m);
      d.pending = true;
      m->apply_pending = true;
      d.version = m->slots[src].version + 1;
      if (applied_on) *applied_on = m->slots[src].version;
      m->cur = dst;
      m->slots[src].refs--;
    }
    if (applied) *applied = 1;
    return GA3C_OK;
  }
  if (dtheta) {
    // host gradient: upload and recompute the non-finite flag on the device
    if (cudaMemcpyAsync(c->grad, dtheta, n * sizeof(float), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->flag, 0, sizeof(int), c->stream) != cudaSuccess) {
      unpin();
      set_err("apply_rmsprop: upload failed");
      return GA3C_CUDA_ERROR;
    }
    Launch l(c, GA3C_K_OTHER, -1);
    pdl_launch(c->cur, check_finite_kernel, dim3(kNumSMs), dim3(256), 0, c->grad, n, c->flag);
  }
  c->grad_flag = -1;
  launch_rmsprop(c, m->slots[src], m->slots[dst], nullptr);
  cudaMemcpyAsync(c->h_flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    unpin();
    set_err(std::string("apply_rmsprop: ") + cudaGetErrorString(e));
    return GA3C_CUDA_ERROR;
  }
  {
    // everything this call ordered after has completed
    std::lock_guard<std::mutex> lk(m->read_m);
    m->apply_pending = false;
    for (auto& sl : m->slots) sl.pending = false;
  }
  if (*c->h_flag) {
    unpin();
    if (applied) *applied = 0;
    return GA3C_NOT_APPLIED;
  }
  {
    std::lock_guard<std::mutex> lk(m->read_m);
    m->slots[dst].version = m->slots[src].version + 1;
    if (applied_on) *applied_on = m->slots[src].version;
    m->cur = dst;
    m->slots[src].refs--;
  }
  if (applied) *applied = 1;
  return GA3C_OK;
}

int ga3c_apply_rmsprop_dev(ga3c_ctx* c) {
  if (!c) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  Slot& s = m->slots[m->cur];
  launch_rmsprop(c, s, s, c->dev_version);
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

int ga3c_model_ring(ga3c_model* m, int n, int* slots_out) {
  if (!m || n < 1 || !slots_out) return GA3C_INVALID_ARGUMENT;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  std::lock_guard<std::mutex> uk(m->update_m);
  std::lock_guard<std::mutex> lk(m->read_m);
  const Slot latest = m->slots[m->cur];
  const std::size_t bytes = m->lo.total * sizeof(float);
  for (int i = 0; i < n; ++i) {
    Slot s;
    GA3C_CUDA(cudaMalloc(&s.theta, bytes));
    GA3C_CUDA(cudaMalloc(&s.g, bytes));
    GA3C_CUDA(cudaMemcpy(s.theta, latest.theta, bytes, cudaMemcpyDeviceToDevice));
    GA3C_CUDA(cudaMemcpy(s.g, latest.g, bytes, cudaMemcpyDeviceToDevice));
    s.version = latest.version;
    s.refs = 1;  // owned by the caller's device loop: never recycled
    if (!m->slots.push_back(s)) {
      cudaFree(s.theta);
      cudaFree(s.g);
      set_err("ga3c_model_ring: slot table full");
      return GA3C_OUT_OF_MEMORY;
    }
    slots_out[i] = static_cast<int>(m->slots.size()) - 1;
  }
  return GA3C_OK;
}

int ga3c_apply_rmsprop_slots_dev(ga3c_ctx* c, const ga3c_ctx* grad_from, int src_slot, int dst_slot) {
  if (!c || (grad_from && grad_from->m != c->m) || src_slot < 0 || dst_slot < 0 ||
      src_slot >= (int)c->m->slots.size() || dst_slot >= (int)c->m->slots.size() || src_slot == dst_slot)
    return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  launch_rmsprop(c, m->slots[src_slot], m->slots[dst_slot], c->dev_version, grad_from);
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

// The per-call graphs (tf_graphs) bake the split plans and the stream's
// priority: a context whose budget or priority changes captures them again.
static void drop_call_graphs(ga3c_ctx* c) {
  if (c->tf_graphs.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->tf_graphs) cudaGraphExecDestroy(kv.second);
  c->tf_graphs.clear();
}

int ga3c_ctx_set_sm_budget(ga3c_ctx* c, int sms) {
  if (!c || sms < 0) return GA3C_INVALID_ARGUMENT;
  const int v = std::min(sms, kNumSMs);
  if (v != c->sms) drop_call_graphs(c);
  c->sms = v;
  return GA3C_OK;
}

int ga3c_ctx_set_priority(ga3c_ctx* c, int level) {
  if (!c || level < 0) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  int prio_lo = 0, prio_hi = 0;
  GA3C_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // numerically lower = higher priority; the side streams stay lowest
  const int prio = std::min(prio_hi + level, prio_lo);
  GA3C_CUDA(cudaStreamSynchronize(c->stream));
  drop_call_graphs(c);
  cudaStream_t s = nullptr;
  GA3C_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio));
  cudaStreamDestroy(c->stream);
  c->stream = c->cur = s;
  return GA3C_OK;
}

int ga3c_copy_slot_dev(ga3c_ctx* c, int src_slot, int dst_slot) {
  if (!c || src_slot < 0 || dst_slot < 0 || src_slot >= (int)c->m->slots.size() ||
      dst_slot >= (int)c->m->slots.size())
    return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (src_slot == dst_slot) return GA3C_OK;
  const std::size_t bytes = m->lo.total * sizeof(float);
  const Slot& s = m->slots[src_slot];
  const Slot& d = m->slots[dst_slot];
  GA3C_CUDA(cudaMemcpyAsync(d.theta, s.theta, bytes, cudaMemcpyDeviceToDevice, c->stream));
  GA3C_CUDA(cudaMemcpyAsync(d.g, s.g, bytes, cudaMemcpyDeviceToDevice, c->stream));
  return GA3C_OK;
}

struct ga3c_dp {
  ga3c_model* m = nullptr;
  int rank = 0, world = 1, ctas = 1;
  dpf::Signal* sig = nullptr;
};

ga3c_dp* ga3c_dp_create(ga3c_model* m, int rank, int world, int ctas, int* status) {
  auto fail = [&](int st) -> ga3c_dp* {
    if (status) *status = st;
    return nullptr;
  };
  if (!m || world < 1 || world > dpf::kMaxRanks || rank < 0 || rank >= world || ctas < 1 || ctas > dpf::kMaxCtas)
    return fail(GA3C_INVALID_ARGUMENT);
  if (set_device(m)) return fail(GA3C_CUDA_ERROR);
  auto* dp = new ga3c_dp;
  dp->m = m;
  dp->rank = rank;
  dp->world = world;
  dp->ctas = ctas;
  if (cudaMalloc(&dp->sig, sizeof(dpf::Signal)) != cudaSuccess ||
      cudaMemset(dp->sig, 0, sizeof(dpf::Signal)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    if (dp->sig) cudaFree(dp->sig);
    delete dp;
    m->set_error("ga3c_dp_create: device allocation failed");
    return fail(GA3C_CUDA_ERROR);
  }
  if (status) *status = GA3C_OK;
  return dp;
}

void ga3c_dp_destroy(ga3c_dp* dp) {
  if (!dp) return;
  set_device(dp->m);
  cudaFree(dp->sig);
  delete dp;
}

void* ga3c_dp_signal(ga3c_dp* dp) { return dp ? dp->sig : nullptr; }

int ga3c_dp_check(ga3c_dp* dp) {
  if (!dp) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = dp->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  GA3C_CUDA(cudaDeviceSynchronize());
  int err = 0;
  GA3C_CUDA(cudaMemcpy(&err, &dp->sig->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) {
    set_err("ga3c_dp_apply: a peer never reached a barrier (timed out)");
    return GA3C_CUDA_ERROR;
  }
  return GA3C_OK;
}

int ga3c_model_slot_theta(ga3c_model* m, int slot, float** theta) {
  if (!m || !theta || slot < 0 || slot >= (int)m->slots.size()) return GA3C_INVALID_ARGUMENT;
  *theta = m->slots[slot].theta;
  return GA3C_OK;
}

int ga3c_dp_apply(ga3c_ctx* c, ga3c_dp* dp, const ga3c_ctx* grad_from, int src_slot, int dst_slot,
                  float* const* peer_grads, float* const* peer_theta_dst, void* const* peer_signals) {
  if (!c || !dp || dp->m != c->m || (grad_from && grad_from->m != c->m) || !peer_grads || !peer_theta_dst ||
      !peer_signals || src_slot < 0 || dst_slot < 0 || src_slot >= (int)c->m->slots.size() ||
      dst_slot >= (int)c->m->slots.size() || src_slot == dst_slot)
    return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  const ga3c_ctx* g = grad_from ? grad_from : c;
  dpf::Peers pr{};
  pr.rank = dp->rank;
  pr.world = dp->world;
  for (int q = 0; q < dp->world; ++q) {
    pr.grad[q] = peer_grads[q];
    pr.theta_dst[q] = peer_theta_dst[q];
    pr.sig[q] = static_cast<dpf::Signal*>(peer_signals[q]);
    if (!pr.grad[q] || !pr.theta_dst[q] || !pr.sig[q]) return GA3C_INVALID_ARGUMENT;
  }
  if (pr.grad[dp->rank] != g->grad || pr.theta_dst[dp->rank] != m->slots[dst_slot].theta ||
      pr.sig[dp->rank] != dp->sig)
    return GA3C_INVALID_ARGUMENT;  // this rank's own entries must be its own buffers
  const ga3c_hyper& hp = m->hp;
  dpf::Step st{m->slots[src_slot].theta, m->slots[src_slot].g, m->slots[dst_slot].g, m->lo.total,
               static_cast<float>(hp.alpha), static_cast<float>(1.0 - hp.alpha), static_cast<float>(hp.eta),
               static_cast<float>(hp.eps_rms), hp.grad_clip_norm, c->dev_version};
  Launch l(c, GA3C_K_RMSPROP, -1);
  // plain launch (no PDL): the kernel spins on peers, it must not start early
  dpf::dp_rmsprop_kernel<<<dp->ctas, dpf::kThreads, 0, c->cur>>>(pr, st);
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

int ga3c_ipc_get_handle(const void* dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64) return GA3C_INVALID_ARGUMENT;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)) != cudaSuccess) return GA3C_CUDA_ERROR;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, sizeof(h));
  return GA3C_OK;
}

int ga3c_ipc_open_handle(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return GA3C_INVALID_ARGUMENT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  if (cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return GA3C_CUDA_ERROR;
  return GA3C_OK;
}

int ga3c_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return GA3C_INVALID_ARGUMENT;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? GA3C_OK : GA3C_CUDA_ERROR;
}

int ga3c_ctx_read_dev_version(ga3c_ctx* c, uint64_t* version) {
  if (!c || !version) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  unsigned long long v = 0;
  GA3C_CUDA(cudaMemcpyAsync(&v, c->dev_version, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
  GA3C_CUDA(cudaStreamSynchronize(c->stream));
  *version = v;
  return GA3C_OK;
}

int ga3c_compute_returns_dev(ga3c_ctx* c, const double* d_rewards, const int32_t* d_off, int n_seg,
                             const uint8_t* d_terminal, const double* d_bootstrap, double gamma,
                             double* d_out) {
  if (!c || n_seg < 0) return GA3C_INVALID_ARGUMENT;
  if (!(gamma > 0.0) || gamma > 1.0) return GA3C_INVALID_ARGUMENT;
  if (n_seg == 0) return GA3C_OK;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  {
    Launch l(c, GA3C_K_RETURNS, -1);
    pdl_launch(c->cur, returns_kernel, dim3((n_seg + 127) / 128), dim3(128), 0, d_rewards, d_off, n_seg, d_terminal,
                                                               d_bootstrap, gamma, d_out);
  }
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

int ga3c_compute_returns(ga3c_ctx* c, const double* rewards, const int32_t* off, int n_seg,
                         const uint8_t* terminal, const double* bootstrap, double gamma,
                         double* out) {
  if (!c || n_seg < 1 || !rewards || !off || !terminal || !bootstrap || !out)
    return GA3C_INVALID_ARGUMENT;
  if (!(gamma > 0.0) || gamma > 1.0) return GA3C_INVALID_ARGUMENT;  // returns.cpp:11-12
  if (off[0] != 0) return GA3C_INVALID_ARGUMENT;
  for (int s = 0; s < n_seg; ++s) {
    if (off[s + 1] <= off[s]) return GA3C_INVALID_ARGUMENT;  // empty segment, returns.cpp:10
    if (!terminal[s] && !std::isfinite(bootstrap[s])) return GA3C_NONFINITE_INPUT;
  }
  const int n = off[n_seg];
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(rewards[i])) return GA3C_NONFINITE_INPUT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (set_device(m)) return GA3C_CUDA_ERROR;
  if ((std::size_t)n > c->r_cap) {
    cudaFree(c->r_rew);
    cudaFree(c->r_out);
    c->r_cap = std::max<std::size_t>(n, 1024);
    GA3C_CUDA(cudaMalloc(&c->r_rew, c->r_cap * sizeof(double)));
    GA3C_CUDA(cudaMalloc(&c->r_out, c->r_cap * sizeof(double)));
  }
  if ((std::size_t)n_seg > c->r_seg_cap) {
    cudaFree(c->r_off);
    cudaFree(c->r_term);
    cudaFree(c->r_boot);
    c->r_seg_cap = std::max<std::size_t>(n_seg, 256);
    GA3C_CUDA(cudaMalloc(&c->r_off, (c->r_seg_cap + 1) * sizeof(int32_t)));
    GA3C_CUDA(cudaMalloc(&c->r_term, c->r_seg_cap));
    GA3C_CUDA(cudaMalloc(&c->r_boot, c->r_seg_cap * sizeof(double)));
  }
  GA3C_CUDA(cudaMemcpyAsync(c->r_rew, rewards, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  GA3C_CUDA(cudaMemcpyAsync(c->r_off, off, (n_seg + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  GA3C_CUDA(cudaMemcpyAsync(c->r_term, terminal, n_seg, cudaMemcpyHostToDevice, c->stream));
  GA3C_CUDA(cudaMemcpyAsync(c->r_boot, bootstrap, n_seg * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int rc = ga3c_compute_returns_dev(c, c->r_rew, c->r_off, n_seg, c->r_term, c->r_boot, gamma, c->r_out);
  if (rc) return rc;
  GA3C_CUDA(cudaMemcpyAsync(out, c->r_out, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  GA3C_CUDA(cudaStreamSynchronize(c->stream));
  return GA3C_OK;
}

int ga3c_sample_actions_dev(ga3c_ctx* c, const float* d_pi, const double* d_u, int B, int A,
                            int32_t* d_actions, int action_stride) {
  if (action_stride < 1) action_stride = 1;
  if (!c || B < 0 || A < 1) return GA3C_INVALID_ARGUMENT;
  if (B == 0) return GA3C_OK;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  // the context's own fp64 policy when the caller passes its last output
  const double* pi64 = (d_pi == nullptr || d_pi == c->pi32) ? c->pi64 : nullptr;
  {
    Launch l(c, GA3C_K_SAMPLE, -1);
    pdl_launch(c->cur, sample_kernel, dim3((B + 127) / 128), dim3(128), 0, d_pi, pi64, d_u, B, A, d_actions,
                                                          action_stride);
  }
  GA3C_CUDA(cudaGetLastError());
  return GA3C_OK;
}

int ga3c_ctx_time_kernel(ga3c_ctx* c, int tag, int layer) {
  if (!c || tag < 0 || tag > GA3C_K_ALL) return GA3C_INVALID_ARGUMENT;
  // events are created up front: a graph capture of the bracketed launches
  // must not create them (it records them as event nodes)
  while (tag != GA3C_K_NONE && c->events.size() < 4096) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    c->events.push_back(e);
  }
  c->timed_tag = tag;
  c->timed_layer = layer;
  c->ev_used = 0;
  return GA3C_OK;
}

int ga3c_ctx_kernel_time(ga3c_ctx* c, double* total_ms, uint64_t* launches) {
  if (!c) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  GA3C_CUDA(cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  for (std::size_t i = 0; i + 1 < c->ev_used; i += 2) {
    float ms = 0.0f;
    GA3C_CUDA(cudaEventElapsedTime(&ms, c->events[i], c->events[i + 1]));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = c->ev_used / 2;
  c->ev_used = 0;
  return GA3C_OK;
}

int ga3c_ctx_timeline(ga3c_ctx* c, int cap, double* start_ms, double* end_ms, int* tags, int* layers,
                      int* streams, int* n) {
  if (!c || cap < 0) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  GA3C_CUDA(cudaDeviceSynchronize());
  const int cnt = static_cast<int>(c->ev_used / 2);
  int k = 0;
  for (int i = 0; i < cnt && k < cap; ++i, ++k) {
    float a = 0.f, b = 0.f;
    GA3C_CUDA(cudaEventElapsedTime(&a, c->events[0], c->events[2 * i]));
    GA3C_CUDA(cudaEventElapsedTime(&b, c->events[0], c->events[2 * i + 1]));
    if (start_ms) start_ms[k] = a;
    if (end_ms) end_ms[k] = b;
    const int meta = c->ev_meta[i];
    if (tags) tags[k] = meta & 0xff;
    if (layers) layers[k] = ((meta >> 8) & 0xff) - 1;
    if (streams) streams[k] = meta >> 16;
  }
  if (n) *n = k;
  c->ev_used = 0;
  return GA3C_OK;
}

int ga3c_ctx_graph_begin(ga3c_ctx* c) {
  if (!c || c->capturing) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  GA3C_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  return GA3C_OK;
}

int ga3c_ctx_graph_end(ga3c_ctx* c, int* graph_id) {
  if (!c || !c->capturing) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  c->capturing = false;
  cudaGraph_t g = nullptr;
  GA3C_CUDA(cudaStreamEndCapture(c->stream, &g));
  cudaGraphExec_t ex = nullptr;
  cudaError_t err = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (err != cudaSuccess) {
    set_err(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(err));
    return GA3C_CUDA_ERROR;
  }
  c->graphs.push_back(ex);
  if (graph_id) *graph_id = static_cast<int>(c->graphs.size()) - 1;
  return GA3C_OK;
}

int ga3c_ctx_graph_launch(ga3c_ctx* c, int graph_id) {
  if (!c || graph_id < 0 || graph_id >= static_cast<int>(c->graphs.size())) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  GA3C_CUDA(cudaGraphLaunch(c->graphs[graph_id], c->stream));
  return GA3C_OK;
}

// Trainer step on host buffers with the n-step returns computed on the device
// (returns.cpp:8-26 for every segment, then nnet.cpp:201-291): one upload,
// returns_kernel -> loss/backward kernels on the context stream, scalars back.
// `states` are host states copied to the context buffer, unless `dev_ready`
// is set: then the u8 states already sit in c->d_in in stream order (the
// frame store's gather).
static int loss_grad_segments(ga3c_ctx* c, int slot, const void* states, bool u8, int B,
                              const int32_t* actions, const double* rewards, const int32_t* off,
                              int n_seg, const uint8_t* terminal, const double* bootstrap, double gamma,
                              int apply_clip, double* scalars, double* returns_out, bool dev_ready = false,
                              Stager* sg_in = nullptr, const std::function<void()>& after_flush = {},
                              const void* after_flush_key = nullptr) {
  if (!c || B < 1 || B > c->max_batch || (!states && !dev_ready) || !actions || !rewards || !off || n_seg < 1 ||
      !terminal || !bootstrap || c->pend.active)  // the stage holds an uncollected prediction
    return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (!(gamma > 0.0) || gamma > 1.0 || off[0] != 0 || off[n_seg] != B) return GA3C_INVALID_ARGUMENT;
  for (int s = 0; s < n_seg; ++s) {
    if (off[s + 1] <= off[s]) return GA3C_INVALID_ARGUMENT;
    if (!terminal[s] && !std::isfinite(bootstrap[s])) return GA3C_NONFINITE_INPUT;
  }
  for (int b = 0; b < B; ++b) {
    if (!std::isfinite(rewards[b])) return GA3C_NONFINITE_INPUT;
    if (actions[b] < 0 || actions[b] >= m->lo.n_actions) return GA3C_INVALID_ARGUMENT;
  }
  const std::size_t dim = m->lo.in_dim;
  if (!dev_ready && !u8 && !all_finite(static_cast<const float*>(states), dim * B)) return GA3C_NONFINITE_INPUT;
  if (set_device(m)) return GA3C_CUDA_ERROR;
  if ((std::size_t)B > c->r_cap) {
    cudaFree(c->r_rew);
    cudaFree(c->r_out);
    c->r_cap = std::max<std::size_t>(B, 1024);
    GA3C_CUDA(cudaMalloc(&c->r_rew, c->r_cap * sizeof(double)));
    GA3C_CUDA(cudaMalloc(&c->r_out, c->r_cap * sizeof(double)));
  }
  if ((std::size_t)n_seg > c->r_seg_cap) {
    cudaFree(c->r_off);
    cudaFree(c->r_term);
    cudaFree(c->r_boot);
    c->r_seg_cap = std::max<std::size_t>(n_seg, 256);
    GA3C_CUDA(cudaMalloc(&c->r_off, (c->r_seg_cap + 1) * sizeof(int32_t)));
    GA3C_CUDA(cudaMalloc(&c->r_term, c->r_seg_cap));
    GA3C_CUDA(cudaMalloc(&c->r_boot, c->r_seg_cap * sizeof(double)));
  }
  int s = slot;
  const bool pinned_here = slot < 0;
  if (pinned_here) ga3c_snapshot_acquire(m, &s, nullptr);
  int rc = GA3C_OK;
  const std::size_t bytes = dim * B * (u8 ? 1 : sizeof(float));
  // small inputs packed into the pinned stage: one copy (plus the states)
  Stager own{c};
  Stager& sg = sg_in ? *sg_in : own;
  const int32_t* d_act = sg.put(actions, B);
  const double* d_rew = sg.put(rewards, B);
  const int32_t* d_off = sg.put(off, n_seg + 1);
  const uint8_t* d_term = sg.put(terminal, n_seg);
  const double* d_boot = sg.put(bootstrap, n_seg);
  double* h_scal = scalars ? sg.take<double>(3) : nullptr;
  double* h_ret = returns_out ? sg.take<double>(B) : nullptr;
  int* h_flg = sg.take<int>(1);
  c->grad_flag = -1;
  if (!d_act || !d_rew || !d_off || !d_term || !d_boot || (scalars && !h_scal) || (returns_out && !h_ret) ||
      !h_flg) {
    if (pinned_here) ga3c_snapshot_release(m, s);
    set_err("loss_grad_segments: batch exceeds the context's staging area");
    return GA3C_INVALID_ARGUMENT;
  }
  // the whole device sequence, issued eagerly or captured (see tf_graphs)
  auto issue = [&]() -> bool {
    if ((!dev_ready && cudaMemcpyAsync(c->d_in, states, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) ||
        !sg.flush())
      return false;
    if (after_flush) after_flush();
    {
      Launch l(c, GA3C_K_RETURNS, -1);
      pdl_launch(c->cur, returns_kernel, dim3((n_seg + 127) / 128), dim3(128), 0, d_rew, d_off, n_seg, d_term,
                 d_boot, gamma, c->d_rets);
    }
    run_loss_grad(c, m->slots[s].theta, c->d_in, u8, d_act, c->d_rets, B, apply_clip != 0);
    if (cudaMemcpyAsync(h_flg, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) return false;
    if (scalars &&
        cudaMemcpyAsync(h_scal, c->scal_sum, sizeof(double) * 3, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      return false;
    if (returns_out &&
        cudaMemcpyAsync(h_ret, c->d_rets, sizeof(double) * B, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      return false;
    return true;
  };
  if (dev_ready && sg_in && !c->capturing && c->timed_tag == 0) {
    // frame-store call: replay the captured sequence of this shape and slot
    // (every pointer it bakes -- stage, workspace, theta of the slot, ring --
    // is fixed for the key; the host wrote this call's inputs into the
    // pinned stage at the same offsets above)
    const ga3c_ctx::TfKey key{s, B, n_seg, (scalars ? 1 : 0) | (returns_out ? 2 : 0) | (apply_clip ? 4 : 0),
                              after_flush_key};
    auto it = c->tf_graphs.find(key);
    if (it == c->tf_graphs.end()) {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ex = nullptr;
      bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      const bool issued = ok && issue();
      ok = cudaStreamEndCapture(c->stream, &g) == cudaSuccess && issued && g &&
           cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
      if (!ok) {
        cudaGetLastError();
        if (pinned_here) ga3c_snapshot_release(m, s);
        set_err("loss_grad_segments: graph capture failed");
        return GA3C_CUDA_ERROR;
      }
      it = c->tf_graphs.emplace(key, ex).first;
    }
    wait_slot(c, s);
    if (cudaGraphLaunch(it->second, c->stream) != cudaSuccess) rc = GA3C_CUDA_ERROR;
  } else {
    wait_slot(c, s);
    if (!issue()) rc = GA3C_CUDA_ERROR;
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    rc = GA3C_CUDA_ERROR;
    set_err(std::string("loss_grad_segments: ") + cudaGetErrorString(e));
  }
  if (!rc) c->grad_flag = *h_flg;
  if (!rc && scalars) std::memcpy(scalars, h_scal, sizeof(double) * 3);
  if (!rc && returns_out) std::memcpy(returns_out, h_ret, sizeof(double) * B);
  if (pinned_here) ga3c_snapshot_release(m, s);
  return rc;
}

int ga3c_loss_grad_segments_u8(ga3c_ctx* c, int slot, const uint8_t* frames, int B,
                               const int32_t* actions, const double* rewards,
                               const int32_t* seg_offsets, int n_seg, const uint8_t* terminal,
                               const double* bootstrap, double gamma, int apply_clip,
                               double* scalars, double* returns_out) {
  return loss_grad_segments(c, slot, frames, true, B, actions, rewards, seg_offsets, n_seg, terminal,
                            bootstrap, gamma, apply_clip, scalars, returns_out);
}

// ------------------------------------------------------ frame store
// Device-resident frame stacks: the host sends each
// agent's NEWEST frame (in_h x in_w bytes, 7 KB for 84x84) instead of the
// whole stacked state; the store keeps every agent's last `history` stacked
// states on the device, so the predictor reads its batch and the trainer
// gathers its experiences without another host->device copy.

}  // extern "C"

// pi / v as fp32 (ga3c_predict_frames) or as the fp64 softmax and widened V
// (ga3c_predict_frames64)
template <typename OutT>
static int predict_frames_impl(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                               const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots, OutT* pi,
                               OutT* v, uint64_t* version_used, bool async = false, const double* u = nullptr) {
  constexpr bool f64 = std::is_same<OutT, double>::value;
  if (!c || !f || f->m != c->m) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  if (n < 0 || n > c->max_batch || (n > 0 && (!new_frames || !agents || (!async && (!pi || !v)))) ||
      c->pend.active) {
    set_err("predict_frames: n = " + std::to_string(n) + " (context max_batch " + std::to_string(c->max_batch) +
            (c->pend.active ? "), a prediction of this context is in flight" : "), or a null buffer"));
    return GA3C_INVALID_ARGUMENT;
  }
  std::vector<int32_t> idx(4 * static_cast<std::size_t>(n));
  {
    std::lock_guard<std::mutex> lk(f->mu);
    for (int i = 0; i < n; ++i) {
      const int a = agents[i];
      if (a < 0 || a >= f->n_agents) {
        set_err("predict_frames: agent " + std::to_string(a) + " outside the store's " +
                std::to_string(f->n_agents));
        return GA3C_INVALID_ARGUMENT;
      }
    }
    for (int i = 0; i < n; ++i) {
      const int a = agents[i];
      const bool rst = (resets && resets[i]) || f->count[a] == 0;
      idx[i] = a;
      idx[n + i] = static_cast<int32_t>((f->count[a] + f->history - 1) % f->history);  // source (latest) slot
      idx[2 * n + i] = static_cast<int32_t>(f->count[a] % f->history);                 // destination slot
      idx[3 * n + i] = rst ? 1 : 0;
      f->count[a] += 1;
      if (state_slots) state_slots[i] = idx[2 * n + i];
    }
  }
  if (set_device(m)) return GA3C_CUDA_ERROR;
  int s = slot;
  uint64_t ver = 0;
  const bool pinned_here = slot < 0;
  if (pinned_here) {
    ga3c_snapshot_acquire(m, &s, &ver);
  } else {
    if (slot >= (int)m->slots.size()) {
      set_err("predict_frames: slot " + std::to_string(slot) + " not allocated");
      return GA3C_INVALID_ARGUMENT;
    }
    std::lock_guard<std::mutex> lk(m->read_m);
    ver = m->slots[slot].version;
  }
  int rc = GA3C_OK;
  if (n > 0) {
    // dense stacked states at d_in, the new frames right after them; the
    // index table in, pi and v out through the pinned stage
    uint8_t* dense = static_cast<uint8_t*>(c->d_in);
    uint8_t* newf = dense + static_cast<std::size_t>(c->max_batch) * m->lo.in_dim;
    const int A = m->lo.n_actions;
    Stager sg{c};
    const int32_t* d_idx = sg.put(idx.data(), idx.size());
    const double* d_u = u ? sg.put(u, n) : nullptr;
    OutT* h_pi = sg.take<OutT>(static_cast<std::size_t>(n) * A);
    OutT* h_v = sg.take<OutT>(n);
    int32_t* h_act = u ? sg.take<int32_t>(n) : nullptr;
    if (!d_idx || !h_pi || !h_v || (u && (!d_u || !h_act))) {
      set_err("predict_frames: batch exceeds the context's staging area");
      rc = GA3C_INVALID_ARGUMENT;
    }
    // the caller's frames go up first (their host address changes per call);
    // everything after is the device sequence below
    if (!rc && cudaMemcpyAsync(newf, new_frames, f->frame_px * n, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      rc = GA3C_CUDA_ERROR;
    const void* d_pi = f64 ? static_cast<const void*>(c->pi64) : static_cast<const void*>(c->pi32);
    const void* d_v = f64 ? static_cast<const void*>(c->v64) : static_cast<const void*>(c->v);
    const float* theta = m->slots[s].theta;
    // stage upload -> frame push -> forward -> (device sampling) -> result download
    auto issue = [&]() -> bool {
      if (!sg.flush()) return false;
      {
        Launch l(c, GA3C_K_OTHER, -1);
        pdl_launch(c->cur, frames_push_kernel, dim3((unsigned)((f->frame_px / 4 + 255) / 256), n), dim3(256), 0,
                   reinterpret_cast<uint32_t*>(f->ring), f->frame_px, f->history,
                   reinterpret_cast<const uint32_t*>(newf), d_idx, n, reinterpret_cast<uint32_t*>(dense));
      }
      run_forward(c, theta, dense, true, n);
      if (u) {
        // qac::sample_index on the fp64 policy (util.hpp:46-54) with the
        // caller's uniforms: the action the host would draw, bitwise
        Launch l(c, GA3C_K_SAMPLE, -1);
        pdl_launch(c->cur, sample_kernel, dim3((n + 127) / 128), dim3(128), 0, c->pi32, c->pi64, d_u, n, A,
                   c->d_actions, 1);
      }
      return cudaMemcpyAsync(h_pi, d_pi, sizeof(OutT) * n * A, cudaMemcpyDeviceToHost, c->stream) == cudaSuccess &&
             cudaMemcpyAsync(h_v, d_v, sizeof(OutT) * n, cudaMemcpyDeviceToHost, c->stream) == cudaSuccess &&
             (!u || cudaMemcpyAsync(h_act, c->d_actions, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                                    c->stream) == cudaSuccess);
    };
    if (!rc) {
      wait_slot(c, s);
      if (async && !c->capturing && c->timed_tag == 0) {
        // asynchronous calls (steady agent groups: a few fixed batch shapes)
        // replay the sequence captured for this (slot, batch, outputs, store):
        // every pointer it bakes -- stage offsets, workspace, the slot's
        // theta, the ring -- is fixed for the key, and the host wrote this
        // call's index table and uniforms into the pinned stage at the same
        // offsets (one graph launch instead of ~12 API calls per prediction)
        const ga3c_ctx::TfKey key{s, n, -1, (f64 ? 1 : 0) | (u ? 2 : 0), f->ring};
        auto it = c->tf_graphs.find(key);
        if (it == c->tf_graphs.end()) {
          cudaGraph_t g = nullptr;
          cudaGraphExec_t ex = nullptr;
          bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
          const bool issued = ok && issue();
          ok = cudaStreamEndCapture(c->stream, &g) == cudaSuccess && issued && g &&
               cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
          if (g) cudaGraphDestroy(g);
          if (!ok) {
            cudaGetLastError();
            set_err("predict_frames: graph capture failed");
            rc = GA3C_CUDA_ERROR;
          } else {
            it = c->tf_graphs.emplace(key, ex).first;
          }
        }
        if (!rc && cudaGraphLaunch(it->second, c->stream) != cudaSuccess) rc = GA3C_CUDA_ERROR;
      } else if (!issue()) {
        rc = GA3C_CUDA_ERROR;
      }
    }
    if (async && !rc) {
      // outputs stay in the pinned stage until ga3c_predict_collect64
      if (!c->pend.ev && cudaEventCreateWithFlags(&c->pend.ev, cudaEventDisableTiming) != cudaSuccess)
        rc = GA3C_CUDA_ERROR;
      if (!rc && cudaEventRecord(c->pend.ev, c->stream) != cudaSuccess) rc = GA3C_CUDA_ERROR;
      if (!rc) {
        c->pend.active = true;
        c->pend.h_pi = reinterpret_cast<const double*>(h_pi);
        c->pend.h_v = reinterpret_cast<const double*>(h_v);
        c->pend.h_act = h_act;
        c->pend.n = n;
        c->pend.A = A;
        c->pend.slot = s;
        c->pend.pinned = pinned_here;
        c->pend.ver = ver;
        return GA3C_OK;
      }
    }
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      rc = GA3C_CUDA_ERROR;
      set_err(std::string("predict_frames: ") + cudaGetErrorString(e));
    }
    if (!rc) {
      std::memcpy(pi, h_pi, sizeof(OutT) * n * A);
      std::memcpy(v, h_v, sizeof(OutT) * n);
    }
  }
  if (pinned_here) ga3c_snapshot_release(m, s);
  if (version_used) *version_used = ver;
  return rc;
}

extern "C" {

int ga3c_predict_frames(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                        const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots, float* pi,
                        float* v, uint64_t* version_used) {
  return predict_frames_impl(c, slot, f, new_frames, agents, resets, n, state_slots, pi, v, version_used);
}

int ga3c_predict_frames64(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                          const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots, double* pi,
                          double* v, uint64_t* version_used) {
  return predict_frames_impl(c, slot, f, new_frames, agents, resets, n, state_slots, pi, v, version_used);
}

int ga3c_predict_frames64_async(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                                const int32_t* agents, const uint8_t* resets, int n, int32_t* state_slots) {
  if (n < 1) return GA3C_INVALID_ARGUMENT;
  return predict_frames_impl<double>(c, slot, f, new_frames, agents, resets, n, state_slots, nullptr, nullptr,
                                     nullptr, true);
}

int ga3c_predict_frames_act64_async(ga3c_ctx* c, int slot, ga3c_frames* f, const uint8_t* new_frames,
                                    const int32_t* agents, const uint8_t* resets, int n, const double* u,
                                    int32_t* state_slots) {
  if (n < 1 || !u) return GA3C_INVALID_ARGUMENT;
  return predict_frames_impl<double>(c, slot, f, new_frames, agents, resets, n, state_slots, nullptr, nullptr,
                                     nullptr, true, u);
}

int ga3c_predict_collect_act64(ga3c_ctx* c, int32_t* actions, double* v, double* pi, uint64_t* version_used) {
  if (!c || !c->pend.active || !c->pend.h_act || !actions || !v) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  const cudaError_t e = cudaEventSynchronize(c->pend.ev);
  c->pend.active = false;
  if (c->pend.pinned) ga3c_snapshot_release(m, c->pend.slot);
  if (e != cudaSuccess) {
    set_err(std::string("predict_collect_act64: ") + cudaGetErrorString(e));
    return GA3C_CUDA_ERROR;
  }
  std::memcpy(actions, c->pend.h_act, sizeof(int32_t) * c->pend.n);
  std::memcpy(v, c->pend.h_v, sizeof(double) * c->pend.n);
  if (pi) std::memcpy(pi, c->pend.h_pi, sizeof(double) * c->pend.n * c->pend.A);
  if (version_used) *version_used = c->pend.ver;
  return GA3C_OK;
}

int ga3c_predict_collect64(ga3c_ctx* c, double* pi, double* v, uint64_t* version_used) {
  if (!c || !c->pend.active || !pi || !v) return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  auto set_err = [&](const std::string& e) { m->set_error(e); };
  const cudaError_t e = cudaEventSynchronize(c->pend.ev);
  c->pend.active = false;
  if (c->pend.pinned) ga3c_snapshot_release(m, c->pend.slot);
  if (e != cudaSuccess) {
    set_err(std::string("predict_collect64: ") + cudaGetErrorString(e));
    return GA3C_CUDA_ERROR;
  }
  std::memcpy(pi, c->pend.h_pi, sizeof(double) * c->pend.n * c->pend.A);
  std::memcpy(v, c->pend.h_v, sizeof(double) * c->pend.n);
  if (version_used) *version_used = c->pend.ver;
  return GA3C_OK;
}

int ga3c_train_frames(ga3c_ctx* c, int slot, ga3c_frames* f, const int32_t* agents, const int32_t* state_slots,
                      int B, const int32_t* actions, const double* rewards, const int32_t* seg_offsets, int n_seg,
                      const uint8_t* terminal, const double* bootstrap, double gamma, int apply_clip,
                      double* scalars, double* returns_out) {
  if (!c || !f || f->m != c->m || B < 1 || B > c->max_batch || !agents || !state_slots) return GA3C_INVALID_ARGUMENT;
  for (int b = 0; b < B; ++b)
    if (agents[b] < 0 || agents[b] >= f->n_agents || state_slots[b] < 0 || state_slots[b] >= f->history)
      return GA3C_INVALID_ARGUMENT;
  ga3c_model* m = c->m;
  if (set_device(m)) return GA3C_CUDA_ERROR;
  std::vector<int32_t> idx(2 * static_cast<std::size_t>(B));
  std::copy(agents, agents + B, idx.begin());
  std::copy(state_slots, state_slots + B, idx.begin() + B);
  Stager sg{c};
  const int32_t* d_idx = sg.put(idx.data(), idx.size());
  if (!d_idx) return GA3C_INVALID_ARGUMENT;
  // the gather runs after the single staged copy, before the returns/loss kernels
  return loss_grad_segments(c, slot, nullptr, true, B, actions, rewards, seg_offsets, n_seg, terminal, bootstrap,
                            gamma, apply_clip, scalars, returns_out, true, &sg, [&] {
                              Launch l(c, GA3C_K_OTHER, -1);
                              pdl_launch(c->cur, frames_gather_kernel,
                                         dim3((unsigned)((f->frame_px / 4 + 255) / 256), B), dim3(256), 0,
                                         reinterpret_cast<const uint32_t*>(f->ring), f->frame_px, f->history,
                                         d_idx, B, reinterpret_cast<uint32_t*>(c->d_in));
                            },
                            f->ring);
}

void* ga3c_host_alloc(size_t bytes, int* status) {
  void* p = nullptr;
  if (cudaMallocHost(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) {
    if (status) *status = GA3C_OUT_OF_MEMORY;
    return nullptr;
  }
  if (status) *status = GA3C_OK;
  return p;
}

void ga3c_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

ga3c_frames* ga3c_frames_create(ga3c_model* m, int n_agents, int history, int* status) {
  auto fail = [&](int st) -> ga3c_frames* {
    if (status) *status = st;
    return nullptr;
  };
  if (!m || n_agents < 1 || history < 2) return fail(GA3C_INVALID_ARGUMENT);
  if (m->spec.in_c != 4 || m->lo.in_dim % 16 != 0) return fail(GA3C_INVALID_ARGUMENT);  // 4-frame u8 stacks
  if (set_device(m)) return fail(GA3C_CUDA_ERROR);
  auto* f = new ga3c_frames();
  f->m = m;
  f->n_agents = n_agents;
  f->history = history;
  f->frame_px = static_cast<std::size_t>(m->spec.in_h) * m->spec.in_w;
  f->count.assign(n_agents, 0);
  const std::size_t bytes = static_cast<std::size_t>(n_agents) * history * m->lo.in_dim;
  if (cudaMalloc(&f->ring, bytes) != cudaSuccess || cudaMemset(f->ring, 0, bytes) != cudaSuccess) {
    cudaFree(f->ring);
    delete f;
    return fail(GA3C_OUT_OF_MEMORY);
  }
  if (status) *status = GA3C_OK;
  return f;
}

void ga3c_frames_destroy(ga3c_frames* f) {
  if (!f) return;
  cudaSetDevice(f->m->device);
  cudaFree(f->ring);
  delete f;
}

int ga3c_frames_read(ga3c_frames* f, int agent, int state_slot, uint8_t* state) {
  if (!f || agent < 0 || agent >= f->n_agents || state_slot < 0 || state_slot >= f->history || !state)
    return GA3C_INVALID_ARGUMENT;
  if (set_device(f->m)) return GA3C_CUDA_ERROR;
  const std::size_t dim = f->m->lo.in_dim;
  const cudaError_t e = cudaMemcpy(state, f->ring + (static_cast<std::size_t>(agent) * f->history + state_slot) * dim,
                                   dim, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? GA3C_OK : GA3C_CUDA_ERROR;
}

int ga3c_loss_grad_segments_f32(ga3c_ctx* c, int slot, const float* states, int B,
                                const int32_t* actions, const double* rewards,
                                const int32_t* seg_offsets, int n_seg, const uint8_t* terminal,
                                const double* bootstrap, double gamma, int apply_clip,
                                double* scalars, double* returns_out) {
  return loss_grad_segments(c, slot, states, false, B, actions, rewards, seg_offsets, n_seg, terminal,
                            bootstrap, gamma, apply_clip, scalars, returns_out);
}

}  // extern "C"
