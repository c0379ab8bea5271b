// dp_fused.cuh -- data-parallel trainer step fused into one kernel over peer
// memory: gradient reduce-scatter + (optional global-norm clip) + RMSProp on
// the rank's shard + all-gather of the new parameters, replacing
// NCCL all-reduce(sum) followed by a full RMSProp on every replica
// (SURVEY.md §8e/§8f item 2).
//
// Semantics restated from the reference (nnet.hpp:88-94 summed gradients,
// nnet.cpp:281-289 clip, nnet.cpp:293-312 RMSProp and its non-finite
// reject):
//   d      = sum over ranks q = 0..W-1 of grad_q      (fixed rank order)
//   reject if any component of d is non-finite on ANY rank: nobody updates,
//          the destination slot receives the source parameters unchanged
//   clip   if clip > 0 and ||d||_2 > clip: d *= clip / ||d||_2 (fp64 scale,
//          norm = fixed-order sum of per-rank fixed-order partial sums)
//   g'     = alpha*g + ((1-alpha)*d)*d ; theta' = theta - (eta*d)/sqrt(g'+eps)
//          with the single-GPU kernel's per-op rounding (rms1, kernels.cu)
// Rank r owns the contiguous shard [r*per, (r+1)*per) (per a multiple of 4
// floats): it reads that shard of every peer's gradient over NVLink, applies
// RMSProp to it, keeps its shard of the rms state (ZeRO-1 style: the other
// shards of g in this replica are not maintained) and stores theta' into
// every rank's destination slot.  All replicas end with bit-identical theta.
//
// Synchronisation: a per-rank signal block in device memory, mapped into
// every peer (CUDA IPC).  Three cross-rank barriers per call, each a release
// store of the call's epoch into every peer's slot [rank] and acquire loads
// of its own W slots: 0 = every rank's gradient is complete (entered the
// call), A = every shard is reduced (+ its non-finite flag and sum of
// squares), B = every rank has pushed its theta' shard.  Within a rank the
// last-arriving CTA (arrival counter) publishes.  All CTAs of a call must be
// co-resident (the grid is small).  Traffic per rank: (W-1)/W * 4 B/param
// read + (W-1)/W * 4 B/param written over NVLink -- the all-reduce's volume,
// with RMSProp on 1/W of the parameters and no separate launches.
#pragma once

#include <cstddef>
#include <cstdint>

namespace ga3c {
namespace dpf {

constexpr int kMaxRanks = 8;
constexpr int kMaxCtas = 148;
constexpr int kThreads = 256;

struct Signal {
  unsigned long long epoch;  // completed calls of this rank
  unsigned int count0, countA, countB;
  int nf_local;
  int err;  // set when a barrier timed out (a peer never arrived): the call did nothing reliable
  unsigned long long flag0[kMaxRanks];  // written by rank q: epoch (entered the call)
  unsigned long long flagA[kMaxRanks];  // written by rank q: epoch << 1 | non-finite
  double ssA[kMaxRanks];                // written by rank q: its shard's sum of squares
  unsigned long long flagB[kMaxRanks];  // written by rank q: epoch (theta' pushed)
  double ss_cta[kMaxCtas];              // this rank's per-CTA partial sums of squares
};

struct Peers {
  float* grad[kMaxRanks];       // every rank's gradient buffer (this rank's shard is overwritten by d)
  float* theta_dst[kMaxRanks];  // every rank's destination parameters
  Signal* sig[kMaxRanks];
  int rank, world;
};

struct Step {
  const float* th_src;  // this rank's source parameters
  const float* g_src;   // this rank's rms state (source slot)
  float* g_dst;         // this rank's rms state (destination slot)
  std::size_t n;
  float alpha, oma, eta, eps;
  double clip;
  unsigned long long* version;  // on-device update counter (nullable)
};

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void rms_op(float& th, float& g, float d, float alpha, float oma, float eta,
                                       float eps) {
  const float acc = __fadd_rn(__fmul_rn(alpha, g), __fmul_rn(__fmul_rn(oma, d), d));
  g = acc;
  th = __fsub_rn(th, __fdiv_rn(__fmul_rn(eta, d), __fsqrt_rn(__fadd_rn(acc, eps))));
}

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// thread 0 of the CTA: wait until every rank wrote `want` (after >> shift).
// A peer that never arrives (a rank died, the ranks' call sequences diverged,
// peer memory not coherent) gives up after 2 s: the call sets Signal::err
// (ga3c_dp_check reports it) instead of hanging the GPU.
__device__ __forceinline__ bool wait_all(const unsigned long long* f, int world, unsigned long long want,
                                         int shift) {
  const unsigned long long t0 = now_ns();
  for (int q = 0; q < world; ++q)
    while ((ld_acquire(f + q) >> shift) != want)
      if (now_ns() - t0 > 2000000000ull) return false;
  return true;
}

__global__ void __launch_bounds__(kThreads) dp_rmsprop_kernel(Peers pr, Step s) {
  __shared__ double red[kThreads / 32];
  __shared__ int nf_sh;
  __shared__ double ss_all_sh;
  __shared__ int nf_all_sh;
  __shared__ int bail_sh;
  const int tid = threadIdx.x, G = gridDim.x;
  Signal* me = pr.sig[pr.rank];
  // a previous call timed out: the ranks' epochs no longer agree, so do not
  // wait again (ga3c_dp_check reports the error; the caller falls back)
  if (*reinterpret_cast<volatile int*>(&me->err)) return;
  const unsigned long long ep = *reinterpret_cast<volatile unsigned long long*>(&me->epoch) + 1ull;
  const int W = pr.world;
  std::size_t per = (s.n + W - 1) / W;
  per = (per + 3) & ~static_cast<std::size_t>(3);
  const std::size_t lo = per * pr.rank < s.n ? per * pr.rank : s.n;
  const std::size_t hi = lo + per < s.n ? lo + per : s.n;
  const std::size_t stride = static_cast<std::size_t>(G) * kThreads;
  float* mine = pr.grad[pr.rank];

  // ---- barrier 0: every rank's gradient is complete
  if (tid == 0) {
    __threadfence_system();
    if (atomicAdd(&me->count0, 1u) == static_cast<unsigned>(G * ep) - 1u)
      for (int q = 0; q < W; ++q) st_release(&pr.sig[q]->flag0[pr.rank], ep);
    bail_sh = !wait_all(me->flag0, W, ep, 0);
    if (bail_sh) atomicExch(&me->err, 1);
    nf_sh = 0;
  }
  __syncthreads();
  if (bail_sh) return;

  // ---- phase 1: reduce this rank's shard (fixed rank order), non-finite flag, sum of squares
  double ss = 0.0;
  int nf = 0;
  for (std::size_t i = lo + (static_cast<std::size_t>(blockIdx.x) * kThreads + tid) * 4; i < hi; i += stride * 4) {
    if (i + 4 <= hi) {
      float4 d = __ldcg(reinterpret_cast<const float4*>(pr.grad[0] + i));
      for (int q = 1; q < W; ++q) {
        const float4 e = __ldcg(reinterpret_cast<const float4*>(pr.grad[q] + i));
        d.x += e.x;
        d.y += e.y;
        d.z += e.z;
        d.w += e.w;
      }
      *reinterpret_cast<float4*>(mine + i) = d;
      nf |= !isfinite(d.x) | !isfinite(d.y) | !isfinite(d.z) | !isfinite(d.w);
      ss += static_cast<double>(d.x) * d.x + static_cast<double>(d.y) * d.y + static_cast<double>(d.z) * d.z +
            static_cast<double>(d.w) * d.w;
    } else {
      for (std::size_t j = i; j < hi; ++j) {
        float d = __ldcg(pr.grad[0] + j);
        for (int q = 1; q < W; ++q) d += __ldcg(pr.grad[q] + j);
        mine[j] = d;
        nf |= !isfinite(d);
        ss += static_cast<double>(d) * d;
      }
    }
  }
  // fixed-order CTA reduction
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  if (nf) atomicOr(&nf_sh, 1);
  __syncthreads();

  // ---- barrier A: shards reduced; exchange non-finite flags and sums of squares
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    me->ss_cta[blockIdx.x] = t;
    if (nf_sh) atomicOr(&me->nf_local, 1);
    __threadfence();
    if (atomicAdd(&me->countA, 1u) == static_cast<unsigned>(G * ep) - 1u) {
      __threadfence();
      double tot = 0.0;
      for (int b = 0; b < G; ++b) tot += *reinterpret_cast<volatile double*>(&me->ss_cta[b]);
      const int nfl = *reinterpret_cast<volatile int*>(&me->nf_local);
      me->nf_local = 0;
      for (int q = 0; q < W; ++q) {
        *reinterpret_cast<volatile double*>(&pr.sig[q]->ssA[pr.rank]) = tot;
        __threadfence_system();
        st_release(&pr.sig[q]->flagA[pr.rank], (ep << 1) | static_cast<unsigned long long>(nfl != 0));
      }
    }
    bail_sh = !wait_all(me->flagA, W, ep, 1);
    if (bail_sh) atomicExch(&me->err, 1);
    int nfa = 0;
    double sa = 0.0;
    for (int q = 0; q < W; ++q) {
      nfa |= static_cast<int>(ld_acquire(&me->flagA[q]) & 1ull);
      sa += *reinterpret_cast<volatile double*>(&me->ssA[q]);
    }
    nf_all_sh = nfa;
    ss_all_sh = sa;
  }
  __syncthreads();
  if (bail_sh) return;

  // ---- phase 2: RMSProp on the shard (or pass-through on reject), push theta' to every rank
  const bool reject = nf_all_sh != 0;
  double scale = 1.0;
  if (s.clip > 0.0) {
    const double norm = sqrt(ss_all_sh);
    if (norm > s.clip) scale = s.clip / norm;
  }
  for (std::size_t i = lo + static_cast<std::size_t>(blockIdx.x) * kThreads + tid; i < hi; i += stride) {
    float th = s.th_src[i], g = s.g_src[i];
    if (!reject) {
      float d = mine[i];
      if (scale != 1.0) d = static_cast<float>(static_cast<double>(d) * scale);
      rms_op(th, g, d, s.alpha, s.oma, s.eta, s.eps);
    }
    s.g_dst[i] = g;
    for (int q = 0; q < W; ++q) pr.theta_dst[q][i] = th;
  }
  __syncthreads();

  // ---- barrier B: every rank pushed its shard (this rank's destination is complete)
  if (tid == 0) {
    __threadfence_system();
    if (atomicAdd(&me->countB, 1u) == static_cast<unsigned>(G * ep) - 1u) {
      for (int q = 0; q < W; ++q) st_release(&pr.sig[q]->flagB[pr.rank], ep);
      if (!reject && s.version) *s.version += 1ull;
      *reinterpret_cast<volatile unsigned long long*>(&me->epoch) = ep;
    }
    if (!wait_all(me->flagB, W, ep, 0)) atomicExch(&me->err, 1);
  }
  __syncthreads();
}

}  // namespace dpf
}  // namespace ga3c
