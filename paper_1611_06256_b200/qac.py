"""Reference-shaped Python API over the B200 C ABI.

Mirrors the reference's Python surface (proj/bindings/qac_module.cpp:42-124,
proj/tests/python/test_smoke.py) for the hot path: NetworkSpec, Hyperparams,
param_count, init_model, init_rms, forward, policy_entropy,
loss_and_gradients, rmsprop_update and compute_returns keep their names,
argument meaning and error behaviour (ValueError where the reference throws
std::invalid_argument).  Every call runs on the GPU through libga3c_b200.so;
parameters travel as fp32 (the device arithmetic type).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _abi
from ._abi import InvalidArgument


class NetworkSpec:
    """nnet.hpp:14-18, extended with VALID NHWC conv layers.

    NetworkSpec(input_dim, hidden_dims, n_actions) is the reference's MLP;
    NetworkSpec.conv((H, W, C), [(Cout, k, stride), ...], hidden, n_actions)
    adds a conv trunk in front (parameters stored OHWI)."""

    def __init__(self, input_dim: int = 0, hidden_dims: Sequence[int] = (), n_actions: int = 0,
                 in_hwc=None, convs=()):
        self.in_hwc = tuple(in_hwc) if in_hwc is not None else (1, 1, int(input_dim))
        self.convs = [tuple(c) for c in convs]
        self.hidden_dims = list(hidden_dims)
        self.n_actions = int(n_actions)

    @classmethod
    def conv(cls, in_hwc, convs, hidden_dims, n_actions):
        return cls(0, hidden_dims, n_actions, in_hwc=in_hwc, convs=convs)

    @property
    def input_dim(self):
        h, w, c = self.in_hwc
        return h * w * c

    def to_c(self) -> _abi.NetSpec:
        s = _abi.NetSpec()
        if len(self.convs) > _abi.MAX_CONV or len(self.hidden_dims) > _abi.MAX_HIDDEN:
            raise InvalidArgument(_abi.INVALID_ARGUMENT, "too many layers")
        s.in_h, s.in_w, s.in_c = self.in_hwc
        s.n_conv = len(self.convs)
        for i, (co, k, st) in enumerate(self.convs):
            s.conv_out[i], s.conv_k[i], s.conv_stride[i] = co, k, st
        s.n_hidden = len(self.hidden_dims)
        for i, h in enumerate(self.hidden_dims):
            s.hidden[i] = h
        s.n_actions = self.n_actions
        return s

    def key(self):
        return (self.in_hwc, tuple(self.convs), tuple(self.hidden_dims), self.n_actions)


def dnn_a(n_actions: int = 6) -> NetworkSpec:
    """DNN A: Conv16 8x8/4, Conv32 4x4/2, FC256."""
    return NetworkSpec.conv((84, 84, 4), [(16, 8, 4), (32, 4, 2)], [256], n_actions)


def dnn_large(stride: int = 1, n_actions: int = 6) -> NetworkSpec:
    """Larger DNN: Conv32 8x8/s, Conv32 4x4/2, Conv64 4x4/2, FC256."""
    return NetworkSpec.conv((84, 84, 4), [(32, 8, stride), (32, 4, 2), (64, 4, 2)], [256], n_actions)


@dataclass
class Hyperparams:
    """nnet.hpp:20-31 (same defaults)."""
    gamma: float = 0.99
    t_max: int = 5
    beta: float = 0.01
    eps_log: float = 1e-6
    eta: float = 3e-4
    alpha: float = 0.99
    eps_rms: float = 1e-8
    value_loss_weight: float = 0.5
    grad_clip_norm: float = 0.0
    clip_rewards: bool = False

    def to_c(self) -> _abi.HyperC:
        h = _abi.HyperC()
        for f in ("gamma", "beta", "eps_log", "eta", "alpha", "eps_rms", "value_loss_weight",
                  "grad_clip_norm"):
            setattr(h, f, float(getattr(self, f)))
        h.t_max = int(self.t_max)
        h.clip_rewards = int(bool(self.clip_rewards))
        return h

    def key(self):
        return tuple(float(getattr(self, f)) for f in self.__dataclass_fields__)


@dataclass
class ModelState:
    theta: np.ndarray
    version: int = 0


@dataclass
class RmsState:
    g: np.ndarray


@dataclass
class GradientPacket:
    dtheta: np.ndarray
    policy_loss: float = 0.0
    value_loss: float = 0.0
    entropy: float = 0.0
    batch_size: int = 0


@dataclass
class ForwardResult:
    policies: np.ndarray
    values: np.ndarray


@dataclass
class UpdateResult:
    model: ModelState
    rms: RmsState
    applied: bool = False


# ------------------------------------------------------------ device cache

_engines = {}


def _engine(spec: NetworkSpec, hyper: Hyperparams | None, batch: int):
    hyper = hyper or Hyperparams()
    key = (spec.key(), hyper.key())
    e = _engines.get(key)
    if e is None or e[1].max_batch < batch:
        if e is not None:
            e[1].close()
        model = e[0] if e is not None else _abi.Model(spec.to_c(), hyper.to_c())
        ctx = _abi.Context(model, max(batch, 64))
        e = (model, ctx)
        _engines[key] = e
    return e


def _validate(spec: NetworkSpec):
    _abi.check(_abi.lib.ga3c_validate_spec(spec.to_c()), "invalid NetworkSpec")


# ----------------------------------------------------------------- the API

def param_count(spec: NetworkSpec) -> int:
    _validate(spec)
    return int(_abi.lib.ga3c_param_count(spec.to_c()))


def init_model(spec: NetworkSpec, seed: int) -> ModelState:
    """nnet::init_model: the reference's seeded draws, rounded to fp32."""
    _validate(spec)
    P = param_count(spec)
    t32 = np.zeros(P, np.float32)
    _abi.check(_abi.lib.ga3c_init_params(spec.to_c(), seed, None, _abi.ptr(t32)))
    return ModelState(t32, 0)


def init_rms(spec: NetworkSpec) -> RmsState:
    return RmsState(np.zeros(param_count(spec), np.float32))


def _states_array(spec, states):
    if isinstance(states, np.ndarray) and states.dtype == np.uint8:
        return states.reshape(states.shape[0], -1)
    arr = np.asarray(states, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr.reshape(1, -1)
    if arr.size and arr.reshape(arr.shape[0], -1).shape[1] != spec.input_dim:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "nnet: state dimension mismatch")
    return arr.reshape(arr.shape[0], -1).astype(np.float32)


def forward(model: ModelState, spec: NetworkSpec, states) -> ForwardResult:
    """nnet::forward nnet.hpp:81."""
    _validate(spec)
    if isinstance(states, list) and any(len(s) != spec.input_dim for s in states):
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "nnet: state dimension mismatch")
    x = _states_array(spec, states)
    m, ctx = _engine(spec, None, max(1, x.shape[0]))
    if len(model.theta) != m.P:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "forward: theta size does not match spec")
    m.load(model.theta, None, model.version)
    pi, v, _ = ctx.forward(x)
    return ForwardResult(pi, v)


def policy_entropy(policy, eps_log: float) -> float:
    """nnet::policy_entropy nnet.hpp:86 (host helper, fp64)."""
    h = 0.0
    for p in policy:
        if p > 0.0 or eps_log > 0.0:
            h -= p * math.log(p + eps_log)
    return h


def loss_and_gradients(model: ModelState, spec: NetworkSpec, hyper: Hyperparams, states,
                       actions, returns) -> GradientPacket:
    """nnet::loss_and_gradients nnet.hpp:94 (batch given as parallel lists,
    like the reference's Python binding qac_module.cpp:106-115)."""
    _validate(spec)
    _abi.check(_abi.lib.ga3c_validate_hyper(hyper.to_c()), "invalid Hyperparams")
    n = len(states)
    if n == 0:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "loss_and_gradients: empty batch")
    if len(returns) != n or len(actions) != n:
        raise InvalidArgument(_abi.INVALID_ARGUMENT,
                              "loss_and_gradients: returns/experiences length mismatch")
    x = _states_array(spec, states)
    m, ctx = _engine(spec, hyper, n)
    if len(model.theta) != m.P:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "theta size does not match spec")
    m.load(model.theta, None, model.version)
    d, sc = ctx.loss_grad(x, actions, returns)
    return GradientPacket(d, float(sc[0]), float(sc[1]), float(sc[2]), n)


def rmsprop_update(model: ModelState, rms: RmsState, grads: GradientPacket,
                   hyper: Hyperparams, spec: NetworkSpec | None = None) -> UpdateResult:
    """nnet::rmsprop_update nnet.hpp:103 (accumulator first; non-finite
    gradient -> inputs back unchanged with applied = False)."""
    _abi.check(_abi.lib.ga3c_validate_hyper(hyper.to_c()), "invalid Hyperparams")
    P = len(model.theta)
    if len(grads.dtheta) != P or len(rms.g) != P:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "rmsprop_update: size mismatch")
    # the update is elementwise over the flat vector: no network layout needed
    th = np.array(model.theta, np.float32)
    g = np.array(rms.g, np.float32)
    d = np.ascontiguousarray(grads.dtheta, np.float32)
    ap = C.c_int(0)
    h = hyper.to_c()
    rc = _abi.lib.ga3c_rmsprop_flat(C.byref(h), 0, P, th.ctypes.data, g.ctypes.data, d.ctypes.data,
                                    C.byref(ap))
    if rc == _abi.NOT_APPLIED or not ap.value:
        return UpdateResult(ModelState(np.array(model.theta, np.float32), model.version),
                            RmsState(np.array(rms.g, np.float32)), False)
    _abi.check(rc, "rmsprop_update")
    return UpdateResult(ModelState(th, model.version + 1), RmsState(g), True)


def compute_returns(rewards, terminal: bool, bootstrap: float, gamma: float) -> List[float]:
    """returns::compute_returns returns.hpp:31 (fp64, bitwise)."""
    r = np.asarray(rewards, np.float64)
    if r.size == 0:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "compute_returns: empty reward sequence")
    _, ctx = _engine(NetworkSpec(1, [], 2), None, 1)
    out = ctx.compute_returns(r, [0, r.size], [int(bool(terminal))], [float(bootstrap)], gamma)
    return [float(x) for x in out]


# ------------------------------------------------------------ host engine

ENV_KINDS = {"bandit": 0, "catch": 1, "delay_lab": 2, "frame_catch": 3, "frames": 4}


@dataclass
class EnvSpec:
    """envs.hpp EnvSpec + the two pixel environments of the B200 engine."""
    kind: str = "bandit"
    n_contexts: int = 4
    n_actions: int = 4
    grid_size: int = 5
    step_delay_us: int = 500
    episode_len: int = 64
    action_repeat: int = 1

    def input_hwc(self):
        if self.kind in ("frame_catch", "frames"):
            return (84, 84, 4)
        dim = {"bandit": self.n_contexts, "catch": self.grid_size ** 2 + self.grid_size, "delay_lab": 4}[self.kind]
        return (1, 1, dim)

    def action_count(self):
        return {"bandit": self.n_actions, "catch": 3, "delay_lab": 2}.get(self.kind, self.n_actions)


def bandit(n_contexts=4, n_actions=4):
    return EnvSpec("bandit", n_contexts=n_contexts, n_actions=n_actions)


def catch_grid(grid_size=5):
    return EnvSpec("catch", grid_size=grid_size)


def delay_lab(step_delay_us=500, episode_len=64):
    return EnvSpec("delay_lab", step_delay_us=step_delay_us, episode_len=episode_len)


def frame_catch(grid_size=7, n_actions=6, step_delay_us=0):
    return EnvSpec("frame_catch", grid_size=grid_size, n_actions=n_actions, step_delay_us=step_delay_us)


def frames(step_delay_us=0, episode_len=64, n_actions=6):
    return EnvSpec("frames", step_delay_us=step_delay_us, episode_len=episode_len, n_actions=n_actions)


def net_for_env(env: EnvSpec, hidden_dims, convs=()):
    """cli::net_for_env (cli.cpp:161-168): a net whose input/actions fit env."""
    return NetworkSpec(0, hidden_dims, env.action_count(), in_hwc=env.input_hwc(), convs=convs)


@dataclass
class KnobConfig:
    n_agents: int = 1
    n_predictors: int = 2
    n_trainers: int = 2
    pred_batch_max: int = 32
    min_train_batch: int = 1
    train_queue_cap: int = 32
    pred_queue_cap: int = 0


@dataclass
class StopCondition:
    max_updates: int | None = None
    max_seconds: float | None = None
    target_score: float | None = None


@dataclass
class PipelineOptions:
    net: NetworkSpec = None
    hyper: Hyperparams = field(default_factory=Hyperparams)
    env: EnvSpec = field(default_factory=EnvSpec)
    knobs: KnobConfig = field(default_factory=KnobConfig)
    stop: StopCondition = field(default_factory=StopCondition)
    seed: int = 1
    anneal: bool = False
    anneal_batches: bool = False
    epoch_s: float = 60.0
    limits: tuple = (64, 16, 16)
    metrics_interval_s: float = 1.0
    greedy: bool = False
    sync_after_submit: bool = False
    capture_trajectory: bool = False
    device: int = 0
    device_frames: bool = False  # frame envs: newest frames in, stacks + training states on the GPU
    trainer_sms: int = -1  # SM budget per trainer context (-1 auto, 0 all)
    predictor_sms: int = -1  # SM budget per predictor context (-1 auto, 0 all)


@dataclass
class RunReport:
    total_updates: int
    skipped_updates: int
    total_predictions: int
    total_episodes: int
    wall_time_s: float
    avg_tps: float
    avg_pps: float
    avg_samples_per_s: float
    mean_lag: float
    final_rolling_score: float
    experiences_produced: int
    experiences_trained: int
    experiences_dropped: int
    experiences_left_queued: int
    final_knobs: KnobConfig
    final_version: int
    final_theta: np.ndarray
    theta_trajectory: list
    episode_scores: list
    anneal_history: list
    pred_batch_mean: float


def _run(opt: PipelineOptions, sync: bool) -> RunReport:
    o = _abi.PipelineOpts()
    _abi.lib.ga3c_default_pipeline_opts(o)
    o.net = opt.net.to_c()
    o.hyper = opt.hyper.to_c()
    e = opt.env
    o.env_kind = ENV_KINDS[e.kind]
    o.n_contexts, o.env_actions, o.grid_size = e.n_contexts, e.n_actions, e.grid_size
    o.step_delay_us, o.episode_len, o.action_repeat = e.step_delay_us, e.episode_len, e.action_repeat
    k = opt.knobs
    o.n_agents, o.n_predictors, o.n_trainers = k.n_agents, k.n_predictors, k.n_trainers
    o.pred_batch_max, o.min_train_batch = k.pred_batch_max, k.min_train_batch
    o.train_queue_cap, o.pred_queue_cap = k.train_queue_cap, k.pred_queue_cap
    o.max_updates = opt.stop.max_updates or 0
    o.max_seconds = opt.stop.max_seconds or 0.0
    o.has_target_score = int(opt.stop.target_score is not None)
    o.target_score = opt.stop.target_score or 0.0
    o.seed = opt.seed
    o.anneal, o.anneal_batches, o.epoch_s = int(opt.anneal), int(opt.anneal_batches), opt.epoch_s
    o.max_agents, o.max_predictors, o.max_trainers = opt.limits
    o.metrics_interval_s = opt.metrics_interval_s
    o.greedy, o.sync_after_submit = int(opt.greedy), int(opt.sync_after_submit)
    o.capture_trajectory, o.device = int(opt.capture_trajectory), opt.device
    o.device_frames = int(opt.device_frames)
    o.trainer_sms, o.predictor_sms = opt.trainer_sms, opt.predictor_sms
    P = int(_abi.lib.ga3c_param_count(o.net))
    cap_traj = (opt.stop.max_updates or 0) if opt.capture_trajectory else 0
    theta = np.zeros(P, np.float32)
    traj = np.zeros((max(cap_traj, 1), P), np.float32)
    scores = np.zeros(1 << 16, np.float64)
    ann = (_abi.AnnealEntry * 256)()
    err = C.create_string_buffer(512)
    r = _abi.RunReportC()
    rc = _abi.lib.ga3c_pipeline_run(o, int(sync), r, _abi.ptr(theta), _abi.ptr(traj) if cap_traj else None,
                                     cap_traj, _abi.ptr(scores), scores.size, ann, 256, err, 512)
    _abi.check(rc, err.value.decode())
    fk = KnobConfig(r.final_n_agents, r.final_n_predictors, r.final_n_trainers, r.final_pred_batch_max,
                    r.final_min_train_batch, k.train_queue_cap, k.pred_queue_cap)
    hist = [dict(knobs=KnobConfig(a.n_agents, a.n_predictors, a.n_trainers, a.pred_batch_max, a.min_train_batch),
                 measured_tps=a.measured_tps, accepted=bool(a.accepted)) for a in ann[:min(r.n_anneal, 256)]]
    return RunReport(r.total_updates, r.skipped_updates, r.total_predictions, r.total_episodes, r.wall_time_s,
                     r.avg_tps, r.avg_pps, r.avg_samples_per_s, r.mean_lag, r.final_rolling_score,
                     r.experiences_produced, r.experiences_trained, r.experiences_dropped,
                     r.experiences_left_queued, fk, r.final_version, theta,
                     [traj[i].copy() for i in range(min(r.n_trajectory, cap_traj))],
                     list(scores[:min(r.total_episodes, scores.size)]), hist, r.last_frame_pred_batch_mean)


def run(opt: PipelineOptions) -> RunReport:
    """pipeline::run (pipeline.hpp:122) on the B200 engine."""
    return _run(opt, False)


def train_sync(opt: PipelineOptions) -> RunReport:
    """reference::train_sync (reference.hpp:30): zero-lag single-thread trainer."""
    return _run(opt, True)
