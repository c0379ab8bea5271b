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
    p.add_argument("--loop-seconds", type=float, default=5.0)
    p.add_argument("--e2e-steps", type=int, default=0)
    p.add_argument("--e2e-windows", type=int, default=3)
    p.add_argument("--e2e-trainers", type=int, default=4, help="trainer threads in the e2e leg (0 = serial)")
    # N_P = 1 measured best (DNN A e2e, median of 3 windows: N_P/N_T 1/4 644-665K, 2/4 584-610K, 3/4 514K,
    # 2/6 546K; large s1 1/3 102K, 2/4 99K): more host threads contend for the GIL and the 16 vCPUs
    p.add_argument("--e2e-predictors", type=int, default=1, help="predictor threads in the e2e leg (N_P)")
    p.add_argument("--trainers", type=int, default=3,
                   help="trainer contexts in flight in the device step (N_T, policy lag N_T - 1 updates)")
    p.add_argument("--cpu-seconds", type=float, default=6.0)
    p.add_argument("--probe", default="conv_fwd:0",
                   help="kernel class[:layer] for the roofline probe (auto = largest eager share)")
    p.add_argument("--trainer-sms", type=int, default=0,
                   help="N_T > 1: SMs each trainer context's split-K plans fill (ga3c_ctx_set_sm_budget); "
                        "0 = auto: 3/4 of them when an update is latency-bound (< 50 MFLOP/sample), else all")
    p.add_argument("--pred-sms", type=int, default=-1,
                   help="same for the predictor context (0 = all, -1 = auto: 64 for latency-bound nets)")
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
        args.pred_sms = 64 if small else 0
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
    """Algorithmic HBM bytes per step of each forward-layer class: the layer's
    input (u8 frames for conv1, fp32 activations otherwise) and its fp32
    output, read/written once per launch (weights are negligible)."""
    layers, _ = layer_geometry(net)
    n_fwd = agents * tmax + agents * tmax  # predictor + trainer recompute
    b = {}
    h, w, c = FRAME
    in_bytes = h * w * c  # u8 state
    for li, l in enumerate(layers):
        out = l["N"] * l["P"] * 4
        key = "conv_fwd" if l["kind"] == "conv" else "fc_fwd"
        b[(key, li)] = float(in_bytes + out) * n_fwd
        in_bytes = out
    return b


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

def cpu_leg(net, agents, tmax, tb, seconds):
    """The reference CPU path (fp64 oracle restatement) on all host threads:
    the same GA3C iteration's forward, loss_and_gradients and RMSProp work."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    convs, hidden = NETS[net]
    spec = O.make_spec(FRAME, convs, hidden, N_ACTIONS)
    hp = O.Hyper()
    th = O.init_model(spec, O.derive_seed(1, [O.SEED_MODEL_INIT])).astype(np.float32).astype(np.float64)
    threads = os.cpu_count() or 1
    fb = min(agents, 8)
    frames = O.synthetic_frames(3, fb)
    st = O.frames_to_states(frames)
    acts, rets = O.synthetic_batch(3, fb, N_ACTIONS)
    fwd_rate, n_fwd = O.throughput(spec, hp, th, st, acts, rets, 0, threads, seconds / 2)
    tr_rate, n_tr = O.throughput(spec, hp, th, st, acts, rets, 1, threads, seconds / 2)
    P = th.size
    g = np.zeros(P)
    d = np.full(P, 1e-3)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < min(1.0, seconds / 6) or reps < 1:
        O.rmsprop_update(hp, th, g, d)
        reps += 1
    t_rms = (time.perf_counter() - t0) / reps
    n = agents * tmax
    updates = n // tb
    t_step = n / fwd_rate + n / tr_rate + updates * t_rms  # rmsprop is serialized (pipeline.cpp:40)
    return dict(value=n / t_step, fwd_rate=fwd_rate, train_rate=tr_rate, t_rms=t_rms, threads=threads,
                sample=(f"{net}: {n_fwd} forwards + {n_tr} loss_and_gradients (batch {fb}/thread) on "
                        f"{threads} threads over {seconds:.0f}s, {reps} single-thread rmsprop_update; "
                        f"step = {n} predictions + {n} trained samples + {updates} updates"))


def run_reference(args, rank):
    if rank != 0:
        return
    # bounded: one short warm-up sample, then up to 3 step samples of a few
    # seconds of CPU work each (the whole arm stays within ~a minute)
    seconds = max(1.0, args.cpu_seconds / 2)
    cpu_leg(args.net, args.agents, args.tmax, args.train_batch, 0.5)
    vals = []
    for _ in range(max(1, min(args.steps, 3))):
        r = cpu_leg(args.net, args.agents, args.tmax, args.train_batch, seconds)
        vals.append(r["value"])
    v = float(np.median(vals))
    n = args.agents * args.tmax
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(args, 1),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": r["threads"], "kind": "port",
                         "sample": r["sample"] + f"; median of {len(vals)} step samples"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def config_of(args, world, sets=None):
    n = args.agents * args.tmax
    return {"workload": f"GA3C iteration ({args.net}): {args.tmax} predictor batches of {args.agents} "
                        f"agents + n-step returns + {n // args.train_batch} trainer updates of "
                        f"{args.train_batch} samples (loss/backward + RMSProp) per GPU",
            "net": args.net, "agents_per_gpu": args.agents, "t_max": args.tmax,
            "predictor_batch": args.agents, "min_train_batch": args.train_batch,
            "global_train_batch": args.train_batch * world, "updates_per_step": n // args.train_batch,
            "params": param_count(args.net), "parallelism": f"dp{world}",
            "trainers_in_flight": args.trainers, "policy_lag_updates": args.trainers - 1,
            "predictor_trainer_overlap": args.trainers > 1 and not args.no_overlap,
            "dp_update": (args.dp if world > 1 and args.trainers > 1 else
                          ("nccl" if world > 1 else "none (1 GPU)")),
            "trainer_sm_budget": args.trainer_sms if args.trainers > 1 else 148,
            "predictor_sm_budget": (args.pred_sms if args.trainers > 1 and not args.no_overlap else None),
            "l2": (f"inputs cycled over {sets} sets = {sets * n * FRAME_BYTES / 1e6:.0f} MB > 126 MB L2"
                   if sets else "n/a")}


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

    torch.cuda.set_device(local)
    if world > 1:
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
            loop.dp_update = dp.nccl_update
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
    if args.probe == "auto":
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
    probe_steps = args.steps
    if graphs is not None:
        # the probed kernel timed inside the real step: one more G-step graph,
        # captured with event-record nodes around every launch of the probed
        # kernel class (on the stream it runs on), replayed once after the
        # timed region
        time_kernel(probe[0], probe[1])
        ctx.graph_begin()
        for pos in range(G):
            step(pos, pos)
        pg = ctx.graph_end()
        ctx.graph_launch(pg)
        ctx.sync()
        torch.cuda.synchronize()
        probe_steps = G
    probe_ms, probe_n = kernel_time()
    time_kernel("none")
    probe_pass = ("one extra replay of a graph of the timed steps with event nodes around the probed "
                  "kernel's launches" if graphs is not None else "inside the timed region")
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    value = world * n / (ms_step / 1e3)

    hbm, bf16, bf16_sus, peak_src = measured_peaks()
    probed_steps = probe_steps
    w = work[probe] * probed_steps
    # the kernel's bound is the lower roofline: below the ridge (measured bf16
    # peak / measured HBM bandwidth) its arithmetic intensity makes it HBM-bound
    byts = bytes_per_step(args.net, NA, T, TB).get(probe)
    ai = work[probe] / byts if byts else None
    if probe[0] == "rmsprop":
        achieved = w / (probe_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s"}
    elif ai is not None and ai < bf16 * 1e3 / hbm:
        achieved = byts * probed_steps / (probe_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "arithmetic_intensity_flop_per_byte": ai, "ridge_flop_per_byte": bf16 * 1e3 / hbm,
                "tflops_achieved": w / (probe_ms / 1e3) / 1e12, "tflops_frac_of_bf16_peak":
                w / (probe_ms / 1e3) / 1e12 / bf16}
    else:
        achieved = w / (probe_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s"}
        if ai is not None:
            roof.update({"arithmetic_intensity_flop_per_byte": ai, "ridge_flop_per_byte": bf16 * 1e3 / hbm})
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.net, {}).get(f"{probe[0]}[{probe[1]}]" if probe[1] >= 0 else probe[0])
        if tr:
            traffic, traffic_src = tr["bytes_per_launch"], f"{tr['launch']}; {tr['capture']}"
    except (OSError, ValueError, KeyError):
        pass
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": traffic, "traffic_source": traffic_src,
                 "kernel": f"{probe[0]}[layer {probe[1]}]", "launches": probe_n,
                 "avg_launch_us": 1e3 * probe_ms / max(1, probe_n),
                 "share_of_step": probe_ms / (ms_step * probed_steps),
                 "probe_pass": probe_pass,
                 "peak_source": f"{peak_src} ({'HBM copy' if probe[0] == 'rmsprop' else 'cuBLAS bf16 burst'})"})

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(args, ctx, model, frames, uni, rewards, terminal, hyper, sets, world, grad_view,
                      stream, dist)

    loop = None
    if rank == 0 and world == 1 and not args.no_loop and args.net == "dnn_a":
        loop = loop_leg(args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_leg(args.net, NA, T, TB, args.cpu_seconds)
        cpu = {"value": r["value"], "unit": "samples/s", "cores": r["threads"], "kind": "port",
               "sample": r["sample"]}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (u8 84x84x4 frames, seeded weights)",
            "config": config_of(args, world, sets),
            "pps": value, "tps_updates_per_s": updates / (ms_step / 1e3),
            "fwd_mflop_per_prediction": fwd_flops_per_sample(args.net) / 1e6,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "ga3c_loop": loop, "gpu_launches": launches,
            "clocks": clk, "kernel_breakdown_ms_per_step": breakdown,
            "cuda_graph": graphs is not None, "steps_per_graph": G if graphs is not None else None,
            "graph_note": graph_note, "dp_fallback": getattr(args, "dp_fallback", None),
            "theta_fingerprint": theta_fingerprint,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def loop_leg(args):
    """BASELINE configs[1] as the reference runs it: the C++ host engine
    (ga3c_pipeline_run = qac::run, pipeline.cpp:100-611) with agent threads
    stepping synthetic 84x84x4 frame environments (envs.cpp Frames, no step
    delay), N_P predictor threads batching the prediction queue into
    ga3c_forward_u8, N_T trainer threads coalescing >= min_train_batch
    experiences into ga3c_loss_grad_segments_u8 + ga3c_apply_rmsprop.  Whole
    28 KB states cross PCIe both ways (the reference's data path); the knobs
    are the paper's best DNN A point (N_A = 128, N_P = N_T = 2)."""
    from paper_1611_06256_b200 import qac
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=qac.frames(step_delay_us=0, episode_len=64))
    opt.knobs = qac.KnobConfig(n_agents=args.agents, n_predictors=2, n_trainers=2, pred_batch_max=args.agents,
                               min_train_batch=args.train_batch)
    opt.stop = qac.StopCondition(max_seconds=args.loop_seconds)
    r = qac.run(opt)
    return {"value": r.avg_samples_per_s, "unit": "samples/s", "tps_updates_per_s": r.avg_tps,
            "pps": r.avg_pps, "updates": r.total_updates, "wall_s": r.wall_time_s, "mean_policy_lag": r.mean_lag,
            "knobs": {"n_agents": args.agents, "n_predictors": 2, "n_trainers": 2,
                      "pred_batch_max": args.agents, "min_train_batch": args.train_batch},
            "path": "C++ host engine (ga3c_pipeline_run): agent threads + prediction/training queues + "
                    "ga3c_forward_u8 / ga3c_loss_grad_segments_u8 / ga3c_apply_rmsprop"}


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
            pi, v, sl, _ = _abi.predict_frames(ctx, store, newf[s][t], agents, prev_term if t == 0 else None)
            slots[:, t] = sl
            cdf = np.cumsum(pi.astype(np.float64), 1)
            hit = u_h[s, t][:, None] < cdf
            a = hit.argmax(1)
            a[~hit.any(1)] = N_ACTIONS - 1
            acts[:, t] = a
        boot = v.astype(np.float64)
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
        d2h = T * NA * (N_ACTIONS + 1 + 1) * 4 + updates * (3 * 8 + TB * 8 + 4)

    def full_state_step(i):
        s = i % hs
        acts = np.zeros((NA, T), np.int32)
        v = None
        for t in range(T):
            pi, v, _ = ctx.forward(fr_time[s][t])
            acts[:, t] = np.minimum((u_h[s, t][:, None] < np.cumsum(pi.astype(np.float64), 1)).argmax(1),
                                    N_ACTIONS - 1)
        rets = ctx.compute_returns(r_h[s].reshape(-1), off, term_h[s], v.astype(np.float64), hyper.gamma)
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
    # half-written model).
    import queue
    import threading
    ctx_t = [_abi.Context(model, max(NA, TB)) for _ in range(args.e2e_trainers)]
    # trainer threads share the GPU like the device step's trainer contexts:
    # the same SM budget rule (e2e 550K -> 574K samples/s for DNN A)
    e2e_sms = int(os.environ.get("GA3C_E2E_SMS", 0)) or (111 if 2.5 * fwd_flops_per_sample(args.net) < 50e6 else 148)
    for c_ in ctx_t:
        c_.set_sm_budget(e2e_sms)
    store.close()
    # training queue of train_queue_cap = 16 segments-batches (the
    # reference's knob, knobs.hpp:15, default 32): the predictor runs up to
    # two steps ahead of the oldest update still training (one step queued,
    # one being predicted), three if a trainer thread stalls while the
    # others drain a whole step, so the store keeps four steps of stacks
    store = _abi.Frames(model, NA, 4 * T + 2)
    q = queue.Queue(maxsize=updates)

    def trainer(j):
        c = ctx_t[j]
        while True:
            item = q.get()
            if item is None:
                q.task_done()
                q.put(None)
                return
            s, acts, slots, boot, u = item
            sl = slice(u * per_upd, (u + 1) * per_upd)
            _abi.train_frames(c, store, np.repeat(agents[sl], T), slots[sl].reshape(-1), acts[sl].reshape(-1),
                              r_h[s][sl].reshape(-1), seg_off, term_h[s][sl], boot[sl], hyper.gamma)
            c.apply_rmsprop()
            q.task_done()

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
                                               pt[gs] if t == 0 else None)
            slots[gs, t] = sl
            cdf = np.cumsum(pi.astype(np.float64), 1)
            hit = u_h[s, t][gs, None] < cdf
            a = hit.argmax(1)
            a[~hit.any(1)] = N_ACTIONS - 1
            acts[gs, t] = a
        vout[gs] = v

    def predict_step(i, pt):
        s = i % hs
        acts = np.zeros((NA, T), np.int32)
        slots = np.zeros((NA, T), np.int32)
        v = np.zeros(NA, np.float64)
        if NP == 1:  # the main thread is the predictor: no hand-off
            predict_group(0, s, pt, acts, slots, v)
        else:
            for f in [pool.submit(predict_group, g, s, pt, acts, slots, v) for g in range(NP)]:
                f.result()
        return s, acts, slots, v

    dt = dt_serial
    mode = "serial calls"
    win_vals = []
    if world == 1 and args.e2e_trainers > 0:
        ths = [threading.Thread(target=trainer, args=(j,), daemon=True) for j in range(args.e2e_trainers)]
        for th in ths:
            th.start()
        pt = np.zeros(NA, np.uint8)

        def window(steps):
            nonlocal pt
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(steps):
                s, acts, slots, boot = predict_step(i, pt)
                for u in range(updates):
                    q.put((s, acts, slots, boot, u))
                pt = term_h[s].astype(np.uint8)
            q.join()  # every update trained and its apply enqueued
            torch.cuda.synchronize()
            return time.perf_counter() - t0

        window(2)  # warm-up
        # three timed windows of k steps each, the median reported: on the
        # 16-vCPU box single windows of host threads vary by up to 1.5x
        wins = sorted(window(k) for _ in range(args.e2e_windows))
        q.put(None)
        for th in ths:
            th.join()
        dt_thr = wins[len(wins) // 2]
        win_vals = [round(n * k / w) for w in wins]
        if dt_thr < dt:
            dt, mode = dt_thr, f"{NP} predictor threads + {args.e2e_trainers} trainer threads"
    for c in ctx_t:
        c.close()
    store.close()
    out = {"value": world * n * k / dt, "unit": "samples/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": k, "ms_per_step": 1e3 * dt / k, "mode": mode,
           "serial_value": world * n * k / dt_serial, "windows": win_vals,
           "timing": f"threaded: median of {len(win_vals)} windows of {k} steps" if win_vals else "serial",
           "path": "ga3c_predict_frames (newest 84x84 frame per agent) / host sampling / ga3c_train_frames / "
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
