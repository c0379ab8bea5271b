#!/usr/bin/env python
"""bench.py -- GA3C hot path (arXiv 1611.06256) on B200.

A STEP is one GA3C iteration of the device-resident hot path for N_A agents
per GPU (BASELINE.json configs[1] minus the CPU
environments):
  t_max predictor batches      forward(N_A frames) + inverse-CDF sampling
                               (pipeline.cpp:65-93, util.hpp:46-54)
  n-step returns               for the N_A agent segments (returns.cpp:8-26),
                               bootstrapped with the value just played (G8)
  trainer updates              N_A*t_max/min_train_batch updates, each
                               loss_and_gradients + RMSProp (pipeline.cpp:241-306)
so every experience is predicted once and trained once: training samples/s
== predictions/s.  The metric is training samples/s (TPS in samples, G3);
updates/s and PPS are reported beside it.  Inputs (u8 84x84x4 frames,
uniform draws, rewards) are synthetic and resident in HBM, cycled over
enough sets to exceed the 126 MB L2.  Data parallel (N>1): each rank runs its
own agents (predictors sharded by agent) and every update all-reduces the
summed gradient over NCCL before the identical RMSProp step.

--impl reference times the reference's CPU path on the host cores (the fp64
oracle restatement, oracle/libga3c_oracle.so, all host threads) on the same
config and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NETS = {  # name -> (convs, hidden)
    "dnn_a": ([(16, 8, 4), (32, 4, 2)], [256]),
    "large1": ([(32, 8, 1), (32, 4, 2), (64, 4, 2)], [256]),
    "large2": ([(32, 8, 2), (32, 4, 2), (64, 4, 2)], [256]),
    "large3": ([(32, 8, 3), (32, 4, 2), (64, 4, 2)], [256]),
    "large4": ([(32, 8, 4), (32, 4, 2), (64, 4, 2)], [256]),
}
FRAME = (84, 84, 4)
FRAME_BYTES = 84 * 84 * 4
N_ACTIONS = 6
METRIC = "training samples/s (GA3C TPS in samples; == predictions/s in the balanced loop)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--net", default="dnn_a", choices=sorted(NETS))
    p.add_argument("--agents", type=int, default=128, help="N_A per GPU (PAPER.md:344-348)")
    p.add_argument("--tmax", type=int, default=5)
    p.add_argument("--train-batch", type=int, default=40, help="min_train_batch (PAPER.md:655)")
    p.add_argument("--sets", type=int, default=0, help="input sets cycled (0 = enough to exceed L2)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-loop", action="store_true", help="skip the C++ GA3C loop leg (ga3c_loop)")
    p.add_argument("--loop-seconds", type=float, default=10.0)
    p.add_argument("--e2e-steps", type=int, default=0)
    p.add_argument("--e2e-windows", type=int, default=7)
    p.add_argument("--e2e-trainers", type=int, default=4, help="trainer threads in the e2e leg (0 = serial)")
    # N_P = 1 measured best (DNN A e2e, median of 3 windows: N_P/N_T 1/4 644-665K, 2/4 584-610K, 3/4 514K,
    # 2/6 546K; large s1 1/3 102K, 2/4 99K): more host threads contend for the GIL and the 16 vCPUs
    p.add_argument("--e2e-predictors", type=int, default=1, help="predictor threads in the e2e leg (N_P)")
    p.add_argument("--e2e-groups", type=int, default=2,
                   help="agent groups one predictor thread keeps in flight (asynchronous predictions)")
    # e2e DNN A, 1 B200, 4 runs: 40 -> 1.010-1.015M, all -> 0.944M samples/s (device step unchanged)
    p.add_argument("--e2e-pred-sms", type=int, default=-1,
                   help="SM budget of the e2e leg's predictor contexts (ga3c_ctx_set_sm_budget; 0 = all, "
                        "-1 = the device step's predictor budget)")
    p.add_argument("--e2e-sampling", default="device", choices=["device", "host"],
                   help="e2e agents' actions: drawn on the device from the agents' uniforms "
                        "(ga3c_predict_frames_act64_async) or on the host from the returned fp64 pi")
    # N_T sweep (DNN A, 1 B200, after the band-staged conv1 weight gradient, two runs each):
    # 4 -> 1.273M, 5 -> 1.279M, 6 -> 1.334M, 8 -> 1.306M samples/s
    p.add_argument("--trainers", type=int, default=6,
                   help="trainer contexts in flight in the device step (N_T, policy lag N_T - 1 updates)")
    p.add_argument("--cpu-seconds", type=float, default=6.0)
    p.add_argument("--probe", default="auto",
                   help="kernel class[:layer] for the headline roofline (auto = the largest in-step share)")
    p.add_argument("--no-large", action="store_true",
                   help="skip the large1 sub-line of the default (dnn_a, 1 GPU) run")
    p.add_argument("--trainer-sms", type=int, default=0,
                   help="N_T > 1: SMs each trainer context's split-K plans fill (ga3c_ctx_set_sm_budget); "
                        "0 = auto: 3/4 of them when an update is latency-bound (< 50 MFLOP/sample), else all")
    p.add_argument("--pred-sms", type=int, default=-1,
                   help="same for the predictor context (0 = all, -1 = auto: 40 for latency-bound nets)")
    p.add_argument("--dp", default="fused", choices=["fused", "nccl"],
                   help="N > 1 with N_T > 1: one fused reduce-scatter + RMSProp + all-gather kernel over NVLink "
                        "peer memory (ga3c_dp_apply), or NCCL all-reduce + RMSProp")
    p.add_argument("--no-overlap", action="store_true",
                   help="N_T > 1: run the predictor phase before the trainers instead of beside them")
    p.add_argument("--no-graph", action="store_true", help="launch eagerly instead of CUDA graphs")
    p.add_argument("--no-graph-warm", action="store_true",
                   help="skip the graph warm-up launches (theta_fingerprint then depends only on W and K)")
    p.add_argument("--graph-steps", type=int, default=0,
                   help="steps chained per CUDA graph (0 = the largest of 8..1 dividing --steps)")
    p.add_argument("--timeline", default="", help="write a per-launch timeline of one eager step here")
    args = p.parse_args()
    # Automatic SM budgets, resolved here so both arms print the same config.
    # Latency-bound updates (DNN A): trainers plan for 3/4 of the SMs, which
    # also puts every ring in shared mode (two CTAs per SM), so the N_T
    # concurrent trainers interleave (sweep: 49 -> 954K, 90..147 ->
    # 978-992K, 148 with deep rings -> 863K samples/s); the predictor beside
    # them plans for a share (all -> 973K, 111 -> 998K, 49..74 -> 1.01M,
    # 16 -> 905K).
    small = 2.5 * fwd_flops_per_sample(args.net) < 50e6
    if args.trainer_sms == 0:
        args.trainer_sms = 111 if small else 148
    if args.pred_sms < 0:
        # N_T = 6 re-sweep (two runs each): 32 -> 1.357M, 40 -> 1.358M, 48 -> 1.353-1.356M,
        # 56 -> 1.337M, 64 -> 1.334M, 96 -> 1.316M samples/s
        args.pred_sms = 40 if small else 0
    if args.e2e_pred_sms < 0:
        args.e2e_pred_sms = args.pred_sms
    return args


# ----------------------------------------------------------------- helpers

def layer_geometry(net):
    convs, hidden = NETS[net]
    h, w, c = FRAME
    layers = []
    for co, k, s in convs:
        oh, ow = (h - k) // s + 1, (w - k) // s + 1
        layers.append(dict(kind="conv", K=k * k * c, N=co, P=oh * ow, params=co * k * k * c + co))
        h, w, c = oh, ow, co
    prev = h * w * c
    for o in hidden:
        layers.append(dict(kind="fc", K=prev, N=o, P=1, params=prev * o + o))
        prev = o
    heads = dict(K=prev, N=N_ACTIONS + 1, params=(prev + 1) * (N_ACTIONS + 1))
    return layers, heads


def param_count(net):
    layers, heads = layer_geometry(net)
    return sum(l["params"] for l in layers) + heads["params"]


def work_per_step(net, agents, tmax, tb):
    """Algorithmic FLOPs (or bytes) per step for each probed kernel class."""
    layers, heads = layer_geometry(net)
    n_fwd = agents * tmax            # states forwarded by the predictors
    n_train = agents * tmax          # samples trained (forward recompute + backward)
    updates = (agents * tmax) // tb
    P = param_count(net)
    w = {}
    for li, l in enumerate(layers):
        mac = l["K"] * l["N"] * l["P"]
        key = "conv_fwd" if l["kind"] == "conv" else "fc_fwd"
        w[(key, li)] = 2.0 * mac * (n_fwd + n_train)
        w[("wgrad", li)] = 2.0 * mac * n_train
        if li > 0:
            w[("dgrad", li)] = 2.0 * mac * n_train
    w[("rmsprop", -1)] = 20.0 * P * updates   # read theta, g, d; write theta, g (fp32)
    return w


def bytes_per_step(net, agents, tmax, tb):
    """Algorithmic HBM bytes per step of each kernel class, every operand
    moved once per launch:
      conv_fwd / fc_fwd[l]  layer input (u8 frames for layer 0, fp32
                            activations otherwise) + fp32 output, per
                            forwarded state (predictor + trainer recompute);
      wgrad[l]              layer input + fp32 output gradient per trained
                            sample, + the fp32 weight gradient per update;
      dgrad[l]              fp32 output gradient in + fp32 input gradient out
                            per trained sample (+ the weights per update);
      rmsprop               theta, g, dtheta read + theta', g' written = 20 B
                            per parameter per update."""
    layers, _ = layer_geometry(net)
    n_train = agents * tmax
    n_fwd = 2 * n_train  # predictor + trainer recompute
    updates = n_train // tb
    b = {}
    h, w, c = FRAME
    in_bytes = h * w * c  # u8 state
    for li, l in enumerate(layers):
        out = l["N"] * l["P"] * 4
        key = "conv_fwd" if l["kind"] == "conv" else "fc_fwd"
        b[(key, li)] = float(in_bytes + out) * n_fwd
        b[("wgrad", li)] = float(in_bytes + out) * n_train + 4.0 * l["params"] * updates
        if li > 0:
            b[("dgrad", li)] = float(out + in_bytes) * n_train + 4.0 * l["params"] * updates
        in_bytes = out
    b[("rmsprop", -1)] = 20.0 * param_count(net) * updates
    return b


# Tensor-core work each kernel class issues per algorithmic FLOP, and the MMA
# kind: 3xTF32 = A_hi*[B_hi|B_lo] + A_lo*B_hi (3 MMA FLOPs per
# FLOP) with the exact-u8 operand skipping A_lo (2); conv1 forward runs the
# exact int8 digits kernel (4 s8 digit MMAs) for predictor batches and the
# 3-piece bf16 kernel for trainer batches -- mixed, charged here as int8.
def issued(key):
    tag, li = key
    if tag == "conv_fwd" and li == 0:
        return "i8", 4.0
    if tag == "wgrad" and li == 0:
        return "tf32", 2.0
    if tag in ("conv_fwd", "fc_fwd", "wgrad", "dgrad"):
        return "tf32", 3.0
    return None, 0.0


def tc_peaks():
    """Dense tcgen05 peaks measured on the box by tools/tc_peak.cu
    (profiles/r2_tc_peaks.json): tf32 / bf16 TFLOP/s and i8 TOP/s."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_tc_peaks.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def kernel_roofline(args, key, ms, launches, steps, ms_step, tc):
    """One kernel class against its own roofline from in-step timings: the
    lower of the measured HBM bandwidth x arithmetic intensity and the
    measured bf16 tensor peak decides the bound; the tensor fraction against
    the peak of the MMA kind the kernel actually issues is reported beside."""
    hbm, bf16, bf16_sus, peak_src = measured_peaks()
    NA, T, TB = args.agents, args.tmax, args.train_batch
    flops = work_per_step(args.net, NA, T, TB)[key] * steps
    byts = bytes_per_step(args.net, NA, T, TB).get(key, 0.0) * steps
    sec = max(ms, 1e-9) / 1e3
    r = {"kernel": f"{key[0]}[layer {key[1]}]", "launches": launches, "avg_launch_us": 1e3 * ms / max(1, launches),
         "share_of_step": ms / (ms_step * steps), "algorithmic_bytes_per_launch": byts / max(1, launches)}
    if key[0] == "rmsprop":
        r.update({"bound": "hbm", "achieved": flops / sec / 1e9, "peak": hbm, "unit": "GB/s"})
    else:
        ai = flops / byts
        r["arithmetic_intensity_flop_per_byte"] = ai
        r["ridge_flop_per_byte"] = bf16 * 1e3 / hbm
        r["tflops_achieved"] = flops / sec / 1e12
        r["tflops_frac_of_bf16_peak"] = r["tflops_achieved"] / bf16
        if ai < bf16 * 1e3 / hbm:
            r.update({"bound": "hbm", "achieved": byts / sec / 1e9, "peak": hbm, "unit": "GB/s"})
        else:
            r.update({"bound": "tensor", "achieved": r["tflops_achieved"], "peak": bf16, "unit": "TFLOP/s"})
        kind, mult = issued(key)
        pk = {"tf32": tc.get("tf32_tflops"), "i8": tc.get("i8_tops"), "bf16": tc.get("bf16_tflops")}.get(kind)
        if kind and pk:
            r["issued_mma"] = kind
            r["issued_tensor_frac"] = r["tflops_achieved"] * mult / pk
    r["frac"] = r["achieved"] / r["peak"]
    r["peak_source"] = f"{peak_src} ({'HBM copy' if r['bound'] == 'hbm' else 'cuBLAS bf16 burst'})"
    traffic, src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.net, {}).get(f"{key[0]}[{key[1]}]" if key[1] >= 0 else key[0])
        if tr:
            traffic, src = tr["bytes_per_launch"], f"{tr['launch']}; {tr['capture']}"
    except (OSError, ValueError, KeyError):
        pass
    r["traffic"], r["traffic_source"] = traffic, src
    return r


def sample_rows(pi, u):
    """qac::sample_index (util.hpp:46-54) per row: the first a with
    u < sum_{<=a} pi accumulated left to right in fp64, else the last action.
    pi is the device's fp64 softmax (ga3c_*64 calls), so this draws exactly
    the action the on-device sampler draws."""
    hit = u[:, None] < np.cumsum(pi, 1)
    a = hit.argmax(1)
    a[~hit.any(1)] = pi.shape[1] - 1
    return a


def fwd_flops_per_sample(net):
    layers, heads = layer_geometry(net)
    return sum(2.0 * l["K"] * l["N"] * l["P"] for l in layers) + 2.0 * heads["K"] * heads["N"]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        util = [float(r[6]) for r in rows if r[6].replace(".", "").isdigit()]
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------- CPU oracle

def cpu_iteration(net, agents, tmax, tb, max_steps, budget_s, warmup=1):
    """The reference's CPU path EXECUTING the same GA3C iteration (not a
    model of it): the fp64 oracle restatement of nnet.cpp / returns.cpp /
    util.hpp (oracle/libga3c_oracle.so, the reference's own code has no conv
    layers) runs t_max predictor forwards of N_A states + sample_index +
    per-agent compute_returns, then N_A*t_max/min_train_batch updates of
    loss_and_gradients + rmsprop_update, with every host thread working on
    each call (rows split across threads: an upper bound on the reference's
    own N_P/N_T thread parallelism).  Steps run until max_steps or budget_s;
    the value is N_A*t_max samples over the median step time."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    convs, hidden = NETS[net]
    spec = O.make_spec(FRAME, convs, hidden, N_ACTIONS)
    hp = O.Hyper()
    th = O.init_model(spec, O.derive_seed(1, [O.SEED_MODEL_INIT])).astype(np.float32).astype(np.float64)
    g = np.zeros_like(th)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(1234)
    n = agents * tmax
    updates = n // tb
    states = rng.integers(0, 256, (agents, tmax) + FRAME, dtype=np.uint8).reshape(agents, tmax, -1) / 256.0
    uni = rng.random((tmax, agents))
    rewards = rng.random((agents, tmax)) * 2 - 1
    terminal = rng.random(agents) < tmax / 64.0

    def one():
        nonlocal th, g
        acts = np.zeros((agents, tmax), np.int32)
        v = None
        for t in range(tmax):
            pi, v = O.forward_mt(spec, th, states[:, t], threads)
            acts[:, t] = sample_rows(pi, uni[t])
        rets = np.stack([O.compute_returns(rewards[a], bool(terminal[a]), 0.0 if terminal[a] else v[a], hp.gamma)
                         for a in range(agents)])
        X, A, R = states.reshape(n, -1), acts.reshape(-1), rets.reshape(-1)
        for u in range(updates):
            sl = slice(u * tb, (u + 1) * tb)
            d, _ = O.loss_and_gradients_mt(spec, hp, th, X[sl], A[sl], R[sl], threads)
            th, g, _ = O.rmsprop_update(hp, th, g, d)

    for _ in range(warmup):
        one()
    times = []
    t_start = time.perf_counter()
    while len(times) < max(1, max_steps) and (not times or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    med = float(np.median(times))
    return dict(value=n / med, threads=threads, steps=len(times), s_per_step=med,
                sample=(f"{net}: {len(times)} executed GA3C iterations ({tmax} x {agents} forwards + sampling + "
                        f"returns, {updates} x (loss_and_gradients on {tb} + rmsprop_update)) on {threads} "
                        f"threads, {med:.2f} s median per step, after {warmup} warm-up step(s)"))


def run_reference(args, rank):
    if rank != 0:
        return
    # bounded: one warm-up step, then up to --steps executed steps within
    # ~60 s of CPU work (the whole arm ends within a few minutes)
    r = cpu_iteration(args.net, args.agents, args.tmax, args.train_batch, args.steps, 60.0,
                      warmup=min(1, args.warmup))
    v = r["value"]
    n = args.agents * args.tmax
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": r["steps"], "warmup": args.warmup, "ms_per_step": 1e3 * n / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(args, int(os.environ.get("WORLD_SIZE", "1"))),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": r["threads"], "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def config_of(args, world):
    """The workload, identical for both arms (no run-specific keys)."""
    from paper_1611_06256_b200.loop import mean_policy_lag
    n = args.agents * args.tmax
    updates = n // args.train_batch
    overlap = args.trainers > 1 and not args.no_overlap
    return {"workload": f"GA3C iteration ({args.net}): {args.tmax} predictor batches of {args.agents} "
                        f"agents + n-step returns + {updates} trainer updates of "
                        f"{args.train_batch} samples (loss/backward + RMSProp) per GPU",
            "net": args.net, "agents_per_gpu": args.agents, "t_max": args.tmax,
            "predictor_batch": args.agents, "min_train_batch": args.train_batch,
            "global_train_batch": args.train_batch * world, "updates_per_step": updates,
            "params": param_count(args.net), "parallelism": f"dp{world}",
            "trainers_in_flight": args.trainers,
            # gradient computed on version U - (N_T - 1), applied on version U
            "gradient_staleness_updates": args.trainers - 1,
            # the reference's lag metric, applied_on - produced_version
            # (pipeline.cpp:289-291), averaged over the step's experiences
            # (paper_1611_06256_b200/loop.py)
            "mean_policy_lag_updates": mean_policy_lag(updates, overlap) if args.trainers > 1
            else (updates - 1) / 2,
            "predictor_trainer_overlap": overlap,
            "dp_update": (args.dp if world > 1 and args.trainers > 1 else
                          ("nccl" if world > 1 else "none (1 GPU)")),
            "trainer_sm_budget": args.trainer_sms if args.trainers > 1 else 148,
            "predictor_sm_budget": (args.pred_sms if overlap else None)}


# ----------------------------------------------------------------- GPU arm

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1611_06256_b200 import _abi

    # test harness only (tests/test_bench_multirank_gpu.py): every rank on
    # cuda:0 over gloo, so the N > 1 path runs on a one-GPU box (NCCL refuses
    # two ranks on one device)
    one_gpu = world > 1 and os.environ.get("GA3C_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    convs, hidden = NETS[args.net]
    spec = _abi.NetSpec()
    spec.in_h, spec.in_w, spec.in_c = FRAME
    spec.n_conv = len(convs)
    for i, (co, k, s) in enumerate(convs):
        spec.conv_out[i], spec.conv_k[i], spec.conv_stride[i] = co, k, s
    spec.n_hidden = len(hidden)
    for i, h in enumerate(hidden):
        spec.hidden[i] = h
    spec.n_actions = N_ACTIONS
    hyper = _abi.default_hyper()
    model = _abi.Model(spec, hyper, device=local)
    NA, T, TB = args.agents, args.tmax, args.train_batch
    n = NA * T
    updates = n // TB
    assert n % TB == 0 and TB % T == 0, "train batch must cover whole agent segments"
    ctx = _abi.Context(model, max(NA, TB))
    P = model.P
    th = np.zeros(P, np.float32)
    _abi.check(_abi.lib.ga3c_init_params(spec, 1 + rank * 0, None, th.ctypes.data))  # identical replicas
    model.load(th)

    # ---- synthetic inputs resident in HBM (agent-major frame rings) ----
    set_bytes = n * FRAME_BYTES
    sets = args.sets or max(2, int(np.ceil(160e6 / set_bytes)))
    sets += sets % 2  # even: the double-buffered experience parity survives the cycle wrap
    g = torch.Generator(device="cuda")
    g.manual_seed(1234 + rank)
    frames = torch.randint(0, 256, (sets, NA, T) + FRAME, dtype=torch.uint8, device="cuda", generator=g)
    uni = torch.rand((sets, T, NA), dtype=torch.float64, device="cuda", generator=g)
    rewards = (torch.rand((sets, NA, T), dtype=torch.float64, device="cuda", generator=g) - 0.5) * 2
    terminal = (torch.rand((sets, NA), device="cuda", generator=g) < T / 64.0).to(torch.uint8)
    offsets = torch.arange(0, n + 1, T, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)

    from paper_1611_06256_b200 import dp
    from paper_1611_06256_b200.loop import GMAX, DeviceLoop, mean_policy_lag
    NT = args.trainers
    loop = DeviceLoop(model, ctx, NA, T, TB, NT, frames, uni, rewards, terminal, trainer_sms=args.trainer_sms,
                      pred_sms=args.pred_sms, overlap=not args.no_overlap, world=world, device=f"cuda:{local}",
                      hyper=hyper)
    grad_view = loop.grad_view
    fused = None
    if world > 1 and NT > 1:
        if args.dp == "fused":
            try:
                fused = dp.FusedUpdate(model, loop.tctx, loop.ring[:loop.R], rank, world)
                fused.self_check(ctx, 0, P, f"cuda:{local}", loop.ring[0], loop.ring[1], loop.ring[2])
            except Exception as e:  # loud: the line records the fallback and why
                print(f"[bench] FUSED DP UPDATE UNAVAILABLE, falling back to NCCL: {e}", file=sys.stderr)
                fused = None
                args.dp = "nccl"
                args.dp_fallback = str(e)
        if fused is not None:
            loop.dp_update = lambda lp, j, U: fused.apply(ctx, j, lp.ring[U % lp.R], lp.ring[(U + 1) % lp.R])
        else:
            loop.nccl = dp.NcclComm(rank, world, local)  # the library's own NCCL entry (ga3c_allreduce_grads)
            loop.dp_update = dp.nccl_update
    elif world > 1:
        loop.nccl = dp.NcclComm(rank, world, local)
    step = loop.step
    time_kernel, kernel_time, launches_all = loop.time_kernel, loop.kernel_time, loop.launches

    def busy():
        # Park the stream behind a ~4 ms spin so the host can enqueue a whole
        # eager step before the GPU reaches it: the probed kernels then run
        # back to back, and their event brackets time the kernels rather than
        # the host's launch rate.
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(8e6))

    # ---- warmup + per-kernel breakdown (untimed) ----
    for i in range(args.warmup):
        step(i)
    ctx.sync()
    breakdown = {}
    probe_keys = sorted(work_per_step(args.net, NA, T, TB))
    for tag in ("conv_fwd", "fc_fwd", "heads", "loss_bwd", "wgrad", "dgrad", "splitk", "rmsprop",
                "returns", "sample", "other"):
        time_kernel(tag, -1)
        busy()
        step(0)
        ms, cnt = kernel_time()
        breakdown[tag] = round(ms, 4)
    for (tag, li) in probe_keys:
        if li >= 0:
            time_kernel(tag, li)
            busy()
            step(0)
            ms, cnt = kernel_time()
            breakdown[f"{tag}[{li}]"] = round(ms, 4)
    time_kernel("none")
    if args.timeline:
        ctx.time_kernel("all")
        busy()
        step(0)
        tl = ctx.timeline()
        time_kernel("none")
        with open(args.timeline, "w") as f:
            f.write("# one eager step, launches queued behind a spin; ms from the first launch\n")
            f.write("# start_ms end_ms dur_us stream kernel[layer]\n")
            for tag, li, sid, a, b in tl:
                f.write(f"{a:9.4f} {b:9.4f} {1e3 * (b - a):8.2f}  s{sid}  {tag}[{li}]\n")
    work = work_per_step(args.net, NA, T, TB)
    if args.probe == "auto":  # eager guess; re-chosen from the in-step timings below
        cand = [(breakdown.get(f"{t}[{l}]" if l >= 0 else t, 0.0), (t, l)) for (t, l) in work]
        probe = max(cand)[1]
    else:
        t, _, l = args.probe.partition(":")
        probe = (t, int(l) if l else -1)
    ctx.sync()
    graphs = None
    G = args.graph_steps or next(g for g in range(GMAX, 0, -1) if args.steps % g == 0)  # steps chained per graph
    assert 1 <= G <= GMAX and args.steps % G == 0, "--graph-steps must divide --steps (and be <= 8)"
    graph_note = None
    if not args.no_graph:
        # one CUDA graph per input set: the whole GA3C iteration replays as a
        # single launch (kernel timing probes are captured as event nodes).
        # The data-parallel exchange is captured too on every rank: the fused
        # kernel is a plain launch and NCCL collectives are capturable.  If
        # the NCCL capture fails, say so and run eagerly.
        try:
            graphs, launches_per_step = loop.capture(G)
        except Exception as e:
            if world == 1 or fused is not None:
                raise
            print(f"[bench] NCCL CAPTURE FAILED, running eagerly: {e}", file=sys.stderr)
            graph_note = f"nccl capture failed: {e}"
            graphs = None
            torch.cuda.synchronize()
    if graphs is not None:
        if not args.no_graph_warm:
            for s in range(sets):  # warm the instantiated graphs
                ctx.graph_launch(graphs[s])
        ctx.sync()
    else:
        time_kernel(probe[0], probe[1])  # eager: probe inside the timed region

    # ---- timed region ----
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.sync()
    l0 = launches_all()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if graphs is not None:
        for i in range(args.steps // G):
            ctx.graph_launch(graphs[i % sets])
    else:
        for i in range(args.steps):
            step(args.warmup + i)
    ev1.record(stream)
    ev1.synchronize()
    ctx.sync()
    launches = launches_all() - l0
    if graphs is not None:
        launches = launches_per_step * args.steps
    ms_total = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if fused is not None:
        fused.dp.check()  # raises if any fused update timed out waiting for a peer
    # fingerprint of the parameters the timed steps produced (every update
    # reads a fixed version, so this is schedule-independent: equal across
    # --graph-steps settings and runs unless a dependency is missing)
    theta_fingerprint = None
    if NT > 1:
        th_now, _ = model.read_slot(loop.latest_slot())
        theta_fingerprint = float(np.abs(th_now.astype(np.float64)).sum())
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    value = world * n / (ms_step / 1e3)

    # ---- every kernel class timed INSIDE the real step ----
    # One more G-step graph per class, captured with event-record nodes
    # around every launch of that class (on the stream it runs on) and
    # replayed once after the timed region; eager (no graphs): the probe
    # brackets ran inside the timed region for the headline class only.
    per_class = {}
    if graphs is not None:
        for key in sorted(work):
            time_kernel(key[0], key[1])
            ctx.graph_begin()
            for pos in range(G):
                step(pos, pos)
            pg = ctx.graph_end()
            ctx.graph_launch(pg)
            ctx.sync()
            torch.cuda.synchronize()
            per_class[key] = kernel_time() + (G,)
            time_kernel("none")
        if args.probe == "auto":
            probe = max(per_class, key=lambda k: per_class[k][0])
    else:
        per_class[probe] = kernel_time() + (args.steps,)
        time_kernel("none")
    probe_pass = ("one extra replay of a graph of the timed steps with event nodes around the class's "
                  "launches" if graphs is not None else "inside the timed region")
    tc = tc_peaks()
    rbk = {f"{k[0]}[{k[1]}]" if k[1] >= 0 else k[0]: kernel_roofline(args, k, *per_class[k], ms_step, tc)
           for k in per_class}
    # concurrent streams overlap the brackets (each includes the contention
    # of the kernels beside it), so shares of the STEP sum above 1; the share
    # of the summed kernel time is what ncu's serialised launch list compares to
    tot = sum(v[0] for v in per_class.values()) or 1.0
    for k, v in per_class.items():
        rbk[f"{k[0]}[{k[1]}]" if k[1] >= 0 else k[0]]["share_of_kernel_time"] = v[0] / tot
    roof = dict(rbk[f"{probe[0]}[{probe[1]}]" if probe[1] >= 0 else probe[0]])
    roof["probe_pass"] = probe_pass
    roof["selection"] = ("auto: the largest in-step share of the step time" if args.probe == "auto"
                         else f"--probe {args.probe}")

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(args, ctx, model, frames, uni, rewards, terminal, hyper, sets, world, grad_view,
                      stream, dist)

    loop_line = None
    if rank == 0 and world == 1 and not args.no_loop and args.net == "dnn_a":
        loop_line = loop_leg(args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_iteration(args.net, NA, T, TB, 1000, args.cpu_seconds)
        cpu = {"value": r["value"], "unit": "samples/s", "cores": r["threads"], "kind": "port",
               "sample": r["sample"]}

    large = None
    if rank == 0 and world == 1 and args.net == "dnn_a" and not args.no_large:
        large = large_leg(args)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (u8 84x84x4 frames, seeded weights)",
            "config": config_of(args, world),
            "l2_flush": f"inputs cycled over {sets} sets = {sets * n * FRAME_BYTES / 1e6:.0f} MB > 126 MB L2",
            "pps": value, "tps_updates_per_s": updates / (ms_step / 1e3),
            "fwd_mflop_per_prediction": fwd_flops_per_sample(args.net) / 1e6,
            "roofline": roof, "roofline_by_kernel": rbk, "tc_peaks_measured": tc or None,
            "cpu_baseline": cpu, "e2e": e2e, "ga3c_loop": loop_line, "gpu_launches": launches,
            "clocks": clk, "kernel_breakdown_ms_per_step": breakdown,
            "cuda_graph": graphs is not None, "steps_per_graph": G if graphs is not None else None,
            "graph_note": graph_note, "dp_fallback": getattr(args, "dp_fallback", None),
            "theta_fingerprint": theta_fingerprint,
            "large1": large,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def large_leg(args):
    """BASELINE configs[2] (the paper's larger DNN at stride 1) measured in the
    same bench invocation: bench.py --net large1 in a child process on this
    GPU, its line embedded (value, e2e, roofline, cpu_baseline, clocks)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--net", "large1", "--steps", "64", "--warmup", "4",
           "--no-loop", "--no-large", "--e2e-steps", "40"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not line:
            return {"error": f"rc {r.returncode}: {r.stderr[-400:]}"}
        d = json.loads(line[-1])
    except (OSError, subprocess.TimeoutExpired, ValueError) as e:
        return {"error": str(e)}
    keep = ("metric", "value", "unit", "ms_per_step", "steps", "warmup", "config", "l2_flush", "pps",
            "tps_updates_per_s", "roofline", "roofline_by_kernel", "cpu_baseline", "e2e", "gpu_launches", "clocks",
            "cuda_graph", "steps_per_graph", "theta_fingerprint")
    d = {k: d.get(k) for k in keep}
    d["command"] = " ".join(cmd[1:])
    return d


def loop_leg(args):
    """BASELINE configs[1]: the C++ host engine (ga3c_pipeline_run = qac::run,
    pipeline.cpp:100-611) on DNN A with agent threads stepping synthetic
    frame environments (envs.cpp Frames, no step delay), predictor threads
    batching the PredictionQueue, trainer threads coalescing >=
    min_train_batch experiences, and the dynamic scheduler running
    (annealer.cpp:28-53, pipeline.cpp:455-476; with the batch-geometry
    extension).  Agents send their newest 84x84 frame; stacks and
    the TrainingQueue's states stay on the GPU (device_frames).  Beside it,
    the reference's data path (whole 28 KB states both ways, fixed knobs at
    the paper's N_A = 128, N_P = N_T = 2)."""
    from paper_1611_06256_b200 import qac
    env = qac.frames(step_delay_us=0, episode_len=64)
    start = qac.KnobConfig(n_agents=2 * args.agents, n_predictors=4, n_trainers=6, pred_batch_max=args.agents,
                           min_train_batch=args.train_batch)
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=env, device_frames=True)
    opt.knobs = start
    opt.anneal, opt.anneal_batches = True, True
    opt.epoch_s = max(0.5, args.loop_seconds / 10)
    opt.limits = (2 * args.agents, 8, 8)
    opt.stop = qac.StopCondition(max_seconds=args.loop_seconds)
    r = qac.run(opt)
    hist = [dict(knobs=[h["knobs"].n_agents, h["knobs"].n_predictors, h["knobs"].n_trainers,
                        h["knobs"].pred_batch_max, h["knobs"].min_train_batch],
                 updates_per_s=round(h["measured_tps"], 1), accepted=h["accepted"])
            for h in r.anneal_history]
    ref = qac.PipelineOptions(net=qac.dnn_a(), env=env)
    ref.knobs = qac.KnobConfig(n_agents=args.agents, n_predictors=2, n_trainers=2, pred_batch_max=args.agents,
                               min_train_batch=args.train_batch)
    ref.stop = qac.StopCondition(max_seconds=min(5.0, args.loop_seconds))
    rw = qac.run(ref)
    fk = r.final_knobs
    return {"value": r.avg_samples_per_s, "unit": "samples/s", "tps_updates_per_s": r.avg_tps,
            "pps": r.avg_pps, "updates": r.total_updates, "wall_s": r.wall_time_s, "mean_policy_lag": r.mean_lag,
            "knobs_start": {"n_agents": start.n_agents, "n_predictors": start.n_predictors,
                            "n_trainers": start.n_trainers, "pred_batch_max": start.pred_batch_max,
                            "min_train_batch": start.min_train_batch},
            "knobs_final": {"n_agents": fk.n_agents, "n_predictors": fk.n_predictors, "n_trainers": fk.n_trainers,
                            "pred_batch_max": fk.pred_batch_max, "min_train_batch": fk.min_train_batch},
            "anneal": {"epoch_s": opt.epoch_s, "batches": True, "history": hist},
            "path": "C++ host engine (ga3c_pipeline_run, device_frames): agent threads + prediction/training "
                    "queues + ga3c_predict_frames64 (newest frames, pinned) / ga3c_train_frames / "
                    "ga3c_apply_rmsprop, annealer on",
            "whole_state_reference_path": {
                "value": rw.avg_samples_per_s, "knobs": [args.agents, 2, 2, args.agents, args.train_batch],
                "path": "ga3c_forward64_u8 / ga3c_loss_grad_segments_u8 / ga3c_apply_rmsprop, 28 KB states "
                        "both ways, fixed knobs"}}


def e2e_leg(args, ctx, model, frames, uni, rewards, terminal, hyper, sets, world, grad_view, stream, dist):
    """The same iteration through the public host-buffer C ABI, inputs and
    outputs in pinned host memory, every host<->device copy inside the timed
    region.  Agents send only their newest 84x84 frame (ga3c_predict_frames:
    the 4-frame stack is built in the device frame store, SURVEY.md §8f row
    1); the host samples actions from pi (util.hpp:46-54); trainers call
    ga3c_train_frames (returns on the device, states gathered from the
    store) and ga3c_apply_rmsprop.  The older full-state calls
    (ga3c_forward_u8 / ga3c_loss_grad_u8, 28 KB per state each way) are
    timed too and reported beside it."""
    import torch
    from paper_1611_06256_b200 import _abi
    NA, T, TB = args.agents, args.tmax, args.train_batch
    n = NA * T
    updates = n // TB
    # windows of 100 steps whatever --steps is: the host-threaded leg needs
    # ~0.1 s windows to be stable (10-step windows: 0.57-0.61M vs 0.72M)
    k = args.e2e_steps or 100
    hs = min(sets, 2)
    px = FRAME[0] * FRAME[1]
    # newest frame of every agent at every step: the last channel of the stacked synthetic states
    newf = [frames[s][..., FRAME[2] - 1].transpose(0, 1).reshape(T, NA, px).contiguous().cpu().pin_memory().numpy()
            for s in range(hs)]
    u_h = uni[:hs].cpu().numpy()
    r_h = rewards[:hs].cpu().numpy()
    term_h = terminal[:hs].cpu().numpy()
    store = _abi.Frames(model, NA, T + 2)
    agents = np.arange(NA, dtype=np.int32)
    seg_off = np.arange(0, TB + 1, T, dtype=np.int32)
    per_upd = TB // T
    prev_term = np.zeros(NA, np.uint8)
    h2d = d2h = 0

    def one(i):
        nonlocal h2d, d2h, prev_term
        s = i % hs
        acts = np.zeros((NA, T), np.int32)
        slots = np.zeros((NA, T), np.int32)
        v = None
        for t in range(T):
            pi, v, sl, _ = _abi.predict_frames(ctx, store, newf[s][t], agents, prev_term if t == 0 else None,
                                               fp64=True)
            slots[:, t] = sl
            acts[:, t] = sample_rows(pi, u_h[s, t])
        boot = v
        for u in range(updates):
            sl = slice(u * per_upd, (u + 1) * per_upd)
            _abi.train_frames(ctx, store, np.repeat(agents[sl], T), slots[sl].reshape(-1), acts[sl].reshape(-1),
                              r_h[s][sl].reshape(-1), seg_off, term_h[s][sl], boot[sl], hyper.gamma,
                              apply_clip=world == 1)
            if grad_view is not None:
                with torch.cuda.stream(stream):
                    dist.all_reduce(grad_view)
                ctx.check_grad()  # reject on the summed gradient, identically on every rank
                ctx.clip_grad()
            ctx.apply_rmsprop()
        prev_term = term_h[s].astype(np.uint8)
        h2d = (T * NA * (px + 4 * 4) + NA + updates * (TB * (4 + 4 + 4 + 8) + 4 * (per_upd + 1) + per_upd * 9))
        d2h = T * NA * (8 * N_ACTIONS + 8 + 4) + updates * (3 * 8 + TB * 8 + 4)  # fp64 pi + V, state slot

    def full_state_step(i):
        s = i % hs
        acts = np.zeros((NA, T), np.int32)
        v = None
        for t in range(T):
            pi, v, _ = ctx.forward(fr_time[s][t], fp64=True)
            acts[:, t] = sample_rows(pi, u_h[s, t])
        rets = ctx.compute_returns(r_h[s].reshape(-1), off, term_h[s], v, hyper.gamma)
        for u in range(updates):
            sl = slice(u * TB // T, (u + 1) * TB // T)
            ctx.loss_grad(fr_agent[s][sl].reshape(TB, -1), acts[sl].reshape(-1), rets[u * TB:(u + 1) * TB],
                          apply_clip=world == 1, want_grad=False)
            ctx.apply_rmsprop()

    def timed(fn, steps):
        for i in range(2):
            fn(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(steps):
            fn(i)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        return dt

    dt_serial = timed(one, k)

    # GA3C's own concurrency (pipeline.cpp:65-93, 241-306): a predictor
    # thread serves the agents while trainer threads, each with its own
    # context (stream), train on finished segments and apply to the latest
    # parameters (out-of-place snapshots, so predictions never read a
    # half-written model).  The trainers share the GPU like the device
    # step's trainer contexts: the same SM budget rule.
    e2e_sms = int(os.environ.get("GA3C_E2E_SMS", 0)) or (111 if 2.5 * fwd_flops_per_sample(args.net) < 50e6 else 148)
    store.close()
    # training queue of train_queue_cap = 16 segments-batches (the
    # reference's knob, knobs.hpp:15, default 32): the predictor runs up to
    # two steps ahead of the oldest update still training (one step queued,
    # one being predicted), three if a trainer thread stalls while the
    # others drain a whole step, so the store keeps four steps of stacks
    store = _abi.Frames(model, NA, 4 * T + 2)
    # GA3C's TrainingQueue + trainer threads, native (ga3c_trainer_pool_*):
    # the predictor hands each update's segment batch over and moves on
    pool_t = _abi.TrainerPool(model, store, args.e2e_trainers, max(NA, TB), e2e_sms, queue_cap=updates) \
        if world == 1 and args.e2e_trainers > 0 else None
    # a step's updates go over in one call: update u = agents [u*per_upd, (u+1)*per_upd)
    # (their T-step segments, agent-major), so every per-sample array is the
    # step's (NA, T) array flattened and the segment tables are regular
    ag_all = np.ascontiguousarray(np.repeat(agents, T))
    b_off = np.arange(0, n + 1, TB, dtype=np.int32)
    s_base = np.arange(0, NA + 1, per_upd, dtype=np.int32)
    s_off = np.ascontiguousarray(np.tile(seg_off, updates))

    def submit_step(s, acts, slots, boot):
        pool_t.submit_many(b_off, s_base, ag_all, slots.reshape(-1), acts.reshape(-1), r_h[s].reshape(-1), s_off,
                           term_h[s], boot, hyper.gamma)

    # N_P predictor threads (GA3C's predictors), each with its own context,
    # serving a contiguous group of agents
    NP = max(1, args.e2e_predictors)
    ctx_p = [ctx] + [_abi.Context(model, NA) for _ in range(NP - 1)]
    from paper_1611_06256_b200.dp import shard
    groups = [slice(a0, a1) for a0, a1 in (shard(NA, g, NP) for g in range(NP))]
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=NP)

    def predict_group(g, s, pt, acts, slots, vout):
        gs = groups[g]
        for t in range(T):
            pi, v, sl, _ = _abi.predict_frames(ctx_p[g], store, newf[s][t][gs], agents[gs],
                                               pt[gs] if t == 0 else None, fp64=True)
            slots[gs, t] = sl
            acts[gs, t] = sample_rows(pi, u_h[s, t][gs])
        vout[gs] = v

    # one predictor thread serving G agent groups on G contexts with
    # asynchronous predictions (ga3c_predict_frames64_async / _collect64): a
    # group's next batch is enqueued as soon as its actions are sampled, so
    # the GPU works on one group while the host samples another
    NG = max(1, args.e2e_groups)
    agroups = [slice(a0, a1) for a0, a1 in (shard(NA, g, NG) for g in range(NG))]
    ctx_g = [ctx] + [_abi.Context(model, NA) for _ in range(NG - 1)]
    if args.e2e_pred_sms > 0:
        for c in ctx_g:
            c.set_sm_budget(args.e2e_pred_sms)

    dev_sample = args.e2e_sampling == "device"

    def predict_groups_async(s, pt, acts, slots, vout):
        # acts / slots are (T, NA) here: each group's row slice is contiguous
        def submit(g, t):
            gs = agroups[g]
            if dev_sample:
                _abi.predict_frames_act_async(ctx_g[g], store, newf[s][t][gs], agents[gs], u_h[s, t][gs],
                                              pt[gs] if t == 0 else None, slots=slots[t, gs])
            else:
                slots[t, gs] = _abi.predict_frames_async(ctx_g[g], store, newf[s][t][gs], agents[gs],
                                                         pt[gs] if t == 0 else None)
        for g in range(NG):
            submit(g, 0)
        for t in range(T):
            for g in range(NG):
                gs = agroups[g]
                if dev_sample:  # qac::sample_index on the device, bitwise the host draw
                    _, v, _, _ = _abi.predict_collect_act(ctx_g[g], actions=acts[t, gs])
                else:
                    pi, v, _ = _abi.predict_collect(ctx_g[g])
                    acts[t, gs] = sample_rows(pi, u_h[s, t][gs])
                if t + 1 < T:
                    submit(g, t + 1)
                else:
                    vout[gs] = v

    def predict_step(i, pt):
        s = i % hs
        acts = np.zeros((NA, T), np.int32)
        slots = np.zeros((NA, T), np.int32)
        v = np.zeros(NA, np.float64)
        if NP == 1 and NG > 1:
            acts_t = np.zeros((T, NA), np.int32)
            slots_t = np.zeros((T, NA), np.int32)
            predict_groups_async(s, pt, acts_t, slots_t, v)
            acts, slots = acts_t.T, slots_t.T
        elif NP == 1:  # the main thread is the predictor: no hand-off
            predict_group(0, s, pt, acts, slots, v)
        else:
            for f in [pool.submit(predict_group, g, s, pt, acts, slots, v) for g in range(NP)]:
                f.result()
        return s, acts, slots, v

    dt = dt_serial
    mode = "serial calls"
    win_vals = []
    if pool_t is not None:
        pt = np.zeros(NA, np.uint8)

        def window(steps):
            nonlocal pt
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(steps):
                s, acts, slots, boot = predict_step(i, pt)
                submit_step(s, acts, slots, boot)
                pt = term_h[s].astype(np.uint8)
            pool_t.wait()  # every update trained and its apply enqueued
            torch.cuda.synchronize()
            return time.perf_counter() - t0

        window(2)  # warm-up
        # seven timed windows of k steps each (~70 ms each), the median reported: on the
        # 16-vCPU box single windows of host threads vary by up to 1.5x
        wins = sorted(window(k) for _ in range(args.e2e_windows))
        dt_thr = wins[len(wins) // 2]
        win_vals = [round(n * k / w) for w in wins]
        if dt_thr < dt:
            dt, mode = dt_thr, (f"{NP} predictor thread(s)"
                                + (f" x {NG} agent groups in flight" if NP == 1 and NG > 1 else "")
                                + (f" on {args.e2e_pred_sms}-SM predictor contexts" if args.e2e_pred_sms > 0 else "")
                                + f" + native trainer pool of {args.e2e_trainers} (ga3c_trainer_pool)"
                                + (", actions sampled on the device" if dev_sample and NP == 1 and NG > 1 else ""))
            if dev_sample and NP == 1 and NG > 1:  # the agents' uniforms up, the drawn actions down
                h2d += n * 8
                d2h += n * 4
        pool_t.close()
    if args.e2e_pred_sms > 0:
        ctx.set_sm_budget(0)
    store.close()
    out = {"value": world * n * k / dt, "unit": "samples/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": k, "ms_per_step": 1e3 * dt / k, "mode": mode,
           "serial_value": world * n * k / dt_serial, "windows": win_vals,
           "timing": f"threaded: median of {len(win_vals)} windows of {k} steps" if win_vals else "serial",
           "path": "ga3c_predict_frames[_act64_async] (newest 84x84 frame per agent) / qac::sample_index "
                   "(device with the host's uniforms, or host) / ga3c_train_frames / "
                   "ga3c_apply_rmsprop (host buffers, pinned)"}
    if world == 1:
        fr_agent = [frames[s].cpu().pin_memory().numpy() for s in range(hs)]
        fr_time = [frames[s].transpose(0, 1).contiguous().cpu().pin_memory().numpy() for s in range(hs)]
        off = np.arange(0, n + 1, T, dtype=np.int32)
        kf = max(3, k // 3)
        dtf = timed(full_state_step, kf)
        out["full_state_api"] = {"value": n * kf / dtf, "h2d_bytes_per_step": 2 * n * FRAME_BYTES,
                                 "path": "ga3c_forward_u8 / ga3c_compute_returns / ga3c_loss_grad_u8 / "
                                         "ga3c_apply_rmsprop (whole 28 KB states both ways)"}
    return out


if __name__ == "__main__":
    main()
