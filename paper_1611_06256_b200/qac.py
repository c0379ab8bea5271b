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
    # the update is shape-agnostic: any spec with P parameters can host it
    m, ctx = _engine(spec if spec is not None else _flat_spec_for(P), hyper, 1)
    m.load(model.theta, rms.g, model.version)
    applied, _ = ctx.apply_rmsprop(np.ascontiguousarray(grads.dtheta, np.float32))
    if not applied:
        return UpdateResult(ModelState(np.array(model.theta, np.float32), model.version),
                        RmsState(np.array(rms.g, np.float32)), False)
    th, g, ver = m.read()
    return UpdateResult(ModelState(th, ver), RmsState(g), True)


def _flat_spec_for(P: int) -> NetworkSpec:
    """A head-only spec {d, [], A} has P = (d + 1) * (A + 1) parameters."""
    for A in range(2, 64):
        if P % (A + 1) == 0 and P // (A + 1) >= 2:
            return NetworkSpec(P // (A + 1) - 1, [], A)
    raise InvalidArgument(_abi.INVALID_ARGUMENT, f"no host layout for {P} parameters; pass spec=")


def compute_returns(rewards, terminal: bool, bootstrap: float, gamma: float) -> List[float]:
    """returns::compute_returns returns.hpp:31 (fp64, bitwise)."""
    r = np.asarray(rewards, np.float64)
    if r.size == 0:
        raise InvalidArgument(_abi.INVALID_ARGUMENT, "compute_returns: empty reward sequence")
    _, ctx = _engine(NetworkSpec(1, [], 2), None, 1)
    out = ctx.compute_returns(r, [0, r.size], [int(bool(terminal))], [float(bootstrap)], gamma)
    return [float(x) for x in out]
