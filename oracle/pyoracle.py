"""ctypes face of the CPU checker -- TEST INFRASTRUCTURE ONLY.

Loads oracle/libga3c_oracle.so (fp64 restatement, see ga3c_oracle.h) and, when
present, oracle/_ref/libqac_ref.so (the reference's own nnet.cpp/returns.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libga3c_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqac_ref.so")

MAX_CONV = 4
MAX_HIDDEN = 4


class Spec(C.Structure):
    """orc_spec / ga3c_net_spec (same layout)."""

    _fields_ = [
        ("in_h", C.c_int), ("in_w", C.c_int), ("in_c", C.c_int),
        ("n_conv", C.c_int),
        ("conv_out", C.c_int * MAX_CONV),
        ("conv_k", C.c_int * MAX_CONV),
        ("conv_stride", C.c_int * MAX_CONV),
        ("n_hidden", C.c_int),
        ("hidden", C.c_int * MAX_HIDDEN),
        ("n_actions", C.c_int),
    ]


class Hyper(C.Structure):
    """orc_hyper / ga3c_hyper, defaults = nnet.hpp:20-31."""

    _fields_ = [
        ("gamma", C.c_double), ("t_max", C.c_int), ("beta", C.c_double),
        ("eps_log", C.c_double), ("eta", C.c_double), ("alpha", C.c_double),
        ("eps_rms", C.c_double), ("value_loss_weight", C.c_double),
        ("grad_clip_norm", C.c_double), ("clip_rewards", C.c_int),
    ]

    def __init__(self, **kw):
        d = dict(gamma=0.99, t_max=5, beta=0.01, eps_log=1e-6, eta=3e-4, alpha=0.99,
                 eps_rms=1e-8, value_loss_weight=0.5, grad_clip_norm=0.0, clip_rewards=0)
        d.update(kw)
        super().__init__(**d)


def make_spec(in_hwc, convs=(), hidden=(), n_actions=6):
    """in_hwc: (H, W, C) or an int input_dim (MLP, reference NetworkSpec)."""
    s = Spec()
    if isinstance(in_hwc, int):
        in_hwc = (1, 1, in_hwc)
    s.in_h, s.in_w, s.in_c = in_hwc
    s.n_conv = len(convs)
    for i, (co, k, st) in enumerate(convs):
        s.conv_out[i], s.conv_k[i], s.conv_stride[i] = co, k, st
    s.n_hidden = len(hidden)
    for i, h in enumerate(hidden):
        s.hidden[i] = h
    s.n_actions = n_actions
    return s


def dnn_a():
    """GA3C DNN A: Conv16 8x8/4, Conv32 4x4/2, FC256, 6 actions."""
    return make_spec((84, 84, 4), [(16, 8, 4), (32, 4, 2)], [256], 6)


def dnn_large(stride=1):
    """The paper's larger DNN: Conv32 8x8/s, Conv32 4x4/2, Conv64 4x4/2, FC256."""
    return make_spec((84, 84, 4), [(32, 8, stride), (32, 4, 2), (64, 4, 2)], [256], 6)


_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_F = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_I = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_U64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load_oracle():
    if not os.path.exists(ORACLE_SO):
        build()
    lib = C.CDLL(ORACLE_SO)
    P = C.POINTER
    lib.orc_mix64.restype = C.c_uint64
    lib.orc_mix64.argtypes = [C.c_uint64]
    lib.orc_derive_seed.restype = C.c_uint64
    lib.orc_derive_seed.argtypes = [C.c_uint64, _U64, C.c_int]
    lib.orc_uniforms.argtypes = [C.c_uint64, _D, C.c_size_t]
    lib.orc_mt64.argtypes = [C.c_uint64, _U64, C.c_size_t]
    lib.orc_sample_index.argtypes = [_D, C.c_int, C.c_double]
    lib.orc_argmax_index.argtypes = [_D, C.c_int]
    lib.orc_validate_spec.argtypes = [P(Spec)]
    lib.orc_validate_hyper.argtypes = [P(Hyper)]
    lib.orc_param_count.restype = C.c_size_t
    lib.orc_param_count.argtypes = [P(Spec)]
    lib.orc_input_dim.restype = C.c_size_t
    lib.orc_input_dim.argtypes = [P(Spec)]
    lib.orc_init_model.argtypes = [P(Spec), C.c_uint64, _D]
    lib.orc_forward.argtypes = [P(Spec), _D, _D, C.c_int, _D, _D]
    lib.orc_policy_entropy.restype = C.c_double
    lib.orc_policy_entropy.argtypes = [_D, C.c_int, C.c_double]
    lib.orc_loss_and_gradients.argtypes = [P(Spec), P(Hyper), _D, _D, _I, _D, C.c_int, _D, _D]
    lib.orc_rmsprop_update.argtypes = [P(Hyper), _D, _D, _D, C.c_size_t, _D, _D]
    lib.orc_rmsprop_update_f32.argtypes = [C.c_float, C.c_float, C.c_float, C.c_float,
                                           _F, _F, _F, C.c_size_t, _F, _F]
    lib.orc_compute_returns.argtypes = [_D, C.c_int, C.c_int, C.c_double, C.c_double, _D]
    lib.orc_throughput.restype = C.c_double
    lib.orc_throughput.argtypes = [P(Spec), P(Hyper), _D, _D, _I, _D, C.c_int, C.c_int, C.c_int,
                                   C.c_double, P(C.c_long)]
    return lib


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load_oracle()
    return _lib


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    """The reference's own nnet.cpp/returns.cpp (oracle/_ref), or None."""
    global _ref
    if _ref is None and ref_available():
        r = C.CDLL(REF_SO)
        P = C.POINTER
        r.ref_param_count.restype = C.c_size_t
        r.ref_param_count.argtypes = [C.c_int, _I, C.c_int, C.c_int]
        r.ref_init_model.argtypes = [C.c_int, _I, C.c_int, C.c_int, C.c_uint64, _D]
        r.ref_forward.argtypes = [C.c_int, _I, C.c_int, C.c_int, _D, C.c_size_t, _D, C.c_int, _D, _D]
        r.ref_loss_and_gradients.argtypes = [C.c_int, _I, C.c_int, C.c_int, P(Hyper), _D,
                                             C.c_size_t, _D, _I, _D, C.c_int, _D, _D]
        r.ref_rmsprop_update.argtypes = [P(Hyper), _D, _D, _D, C.c_size_t, _D, _D, C.c_uint64,
                                         P(C.c_uint64)]
        r.ref_compute_returns.argtypes = [_D, C.c_int, C.c_int, C.c_double, C.c_double, _D]
        r.ref_policy_entropy.restype = C.c_double
        r.ref_policy_entropy.argtypes = [_D, C.c_int, C.c_double]
        r.ref_uniforms.argtypes = [C.c_uint64, _D, C.c_size_t]
        r.ref_sample_many.argtypes = [_D, C.c_int, C.c_uint64, C.c_int, _I]
        r.ref_derive_seed.restype = C.c_uint64
        r.ref_derive_seed.argtypes = [C.c_uint64, _U64, C.c_int]
        _ref = r
    return _ref


class OracleError(ValueError):
    """Raised where the reference throws std::invalid_argument."""


# ---------------------------------------------------------------- wrappers

def param_count(spec):
    return int(lib().orc_param_count(C.byref(spec)))


def input_dim(spec):
    return int(lib().orc_input_dim(C.byref(spec)))


def init_model(spec, seed):
    th = np.zeros(param_count(spec), np.float64)
    if lib().orc_init_model(C.byref(spec), seed, th):
        raise OracleError("init_model: invalid spec")
    return th


def forward(spec, theta, states):
    states = np.ascontiguousarray(states, np.float64).reshape(-1, input_dim(spec))
    B = states.shape[0]
    pi = np.zeros((B, spec.n_actions), np.float64)
    v = np.zeros(B, np.float64)
    if lib().orc_forward(C.byref(spec), np.ascontiguousarray(theta, np.float64), states, B, pi, v):
        raise OracleError("forward: invalid input")
    return pi, v


def loss_and_gradients(spec, hyper, theta, states, actions, returns):
    states = np.ascontiguousarray(states, np.float64).reshape(-1, input_dim(spec))
    B = states.shape[0]
    d = np.zeros(param_count(spec), np.float64)
    sc = np.zeros(3, np.float64)
    rc = lib().orc_loss_and_gradients(
        C.byref(spec), C.byref(hyper), np.ascontiguousarray(theta, np.float64), states,
        np.ascontiguousarray(actions, np.int32), np.ascontiguousarray(returns, np.float64), B, d, sc)
    if rc:
        raise OracleError("loss_and_gradients: invalid input")
    return d, sc


def _chunks(B, threads):
    k = max(1, min(threads, B))
    edges = np.linspace(0, B, k + 1).astype(int)
    return [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]


_POOL = None


def _pool():
    """One persistent host thread pool for the *_mt helpers (ctypes releases
    the GIL, so the chunks run in parallel)."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(os.cpu_count() or 1)
    return _POOL


def forward_mt(spec, theta, states, threads=None):
    """forward over row chunks on `threads` host threads; rows are
    independent, so the result equals forward()."""
    states = np.ascontiguousarray(states, np.float64).reshape(-1, input_dim(spec))
    parts = _chunks(states.shape[0], threads or os.cpu_count() or 1)
    res = list(_pool().map(lambda ab: forward(spec, theta, states[ab[0]:ab[1]]), parts))
    return np.concatenate([r[0] for r in res]), np.concatenate([r[1] for r in res])


def loss_and_gradients_mt(spec, hyper, theta, states, actions, returns, threads=None):
    """loss_and_gradients as a sum of per-chunk sums on host threads (the
    batch sum is associative up to fp64 rounding, far below the fp32 parity
    tolerances this is checked against).  No clip (grad_clip_norm must be 0)."""
    assert hyper.grad_clip_norm == 0.0
    states = np.ascontiguousarray(states, np.float64).reshape(-1, input_dim(spec))
    actions = np.ascontiguousarray(actions, np.int32)
    returns = np.ascontiguousarray(returns, np.float64)
    parts = _chunks(states.shape[0], threads or os.cpu_count() or 1)
    res = list(_pool().map(lambda ab: loss_and_gradients(spec, hyper, theta, states[ab[0]:ab[1]],
                                                         actions[ab[0]:ab[1]], returns[ab[0]:ab[1]]), parts))
    return sum(r[0] for r in res), sum(r[1] for r in res)


def rmsprop_update(hyper, theta, g, dtheta):
    P = len(theta)
    to, go = np.zeros(P), np.zeros(P)
    rc = lib().orc_rmsprop_update(C.byref(hyper), np.ascontiguousarray(theta, np.float64),
                                  np.ascontiguousarray(g, np.float64),
                                  np.ascontiguousarray(dtheta, np.float64), P, to, go)
    if rc < 0:
        raise OracleError("rmsprop_update: invalid hyperparameters")
    return to, go, bool(rc)


def rmsprop_update_f32(hyper, theta, g, dtheta):
    """Bitwise model of the CUDA RMSProp kernel (fp32, one rounding per op)."""
    P = len(theta)
    to, go = np.zeros(P, np.float32), np.zeros(P, np.float32)
    alpha = np.float32(hyper.alpha)
    oma = np.float32(1.0 - hyper.alpha)
    rc = lib().orc_rmsprop_update_f32(alpha, oma, np.float32(hyper.eta), np.float32(hyper.eps_rms),
                                      np.ascontiguousarray(theta, np.float32),
                                      np.ascontiguousarray(g, np.float32),
                                      np.ascontiguousarray(dtheta, np.float32), P, to, go)
    return to, go, bool(rc)


def compute_returns(rewards, terminal, bootstrap, gamma):
    r = np.ascontiguousarray(rewards, np.float64)
    out = np.zeros(len(r), np.float64)
    if lib().orc_compute_returns(r, len(r), int(bool(terminal)), float(bootstrap), float(gamma), out):
        raise OracleError("compute_returns: invalid input")
    return out


def uniforms(seed, n):
    out = np.zeros(n, np.float64)
    lib().orc_uniforms(seed, out, n)
    return out


def derive_seed(base, salts):
    s = np.ascontiguousarray(salts, np.uint64)
    return int(lib().orc_derive_seed(base, s, len(s)))


def sample_index(probs, u):
    p = np.ascontiguousarray(probs, np.float64)
    return int(lib().orc_sample_index(p, len(p), float(u)))


def policy_entropy(p, eps):
    p = np.ascontiguousarray(p, np.float64)
    return float(lib().orc_policy_entropy(p, len(p), eps))


def throughput(spec, hyper, theta, states, actions, returns, mode, n_threads, seconds):
    states = np.ascontiguousarray(states, np.float64).reshape(-1, input_dim(spec))
    B = states.shape[0]
    done = C.c_long(0)
    rate = lib().orc_throughput(C.byref(spec), C.byref(hyper), np.ascontiguousarray(theta, np.float64),
                                states, np.ascontiguousarray(actions, np.int32),
                                np.ascontiguousarray(returns, np.float64), B, mode, n_threads,
                                seconds, C.byref(done))
    return rate, done.value


# ------------------------------------------------------- synthetic inputs

SEED_MODEL_INIT = 0x6D6F64656C   # util.hpp:34 kSeedModelInit
SEED_AGENT_RNG = 0x6167656E74    # util.hpp:35 kSeedAgentRng
TAG_FRAMES = 0x6672616D6573      # "frames": synthetic frame stream


def synthetic_frames(seed, B, hwc=(84, 84, 4)):
    """u8 frames, k = mt19937_64(derive_seed(seed,{TAG_FRAMES,i}))() >> 56 per pixel."""
    H, W, Cc = hwc
    n = H * W * Cc
    out = np.zeros((B, H, W, Cc), np.uint8)
    buf = np.zeros(n, np.uint64)
    for i in range(B):
        lib().orc_mt64(derive_seed(seed, [TAG_FRAMES, i]), buf, n)
        out[i] = (buf >> np.uint64(56)).astype(np.uint8).reshape(H, W, Cc)
    return out


def frames_to_states(frames):
    """x = k / 256, exact in fp64/fp32/tf32/bf16."""
    return frames.reshape(frames.shape[0], -1).astype(np.float64) / 256.0


def synthetic_batch(seed, B, n_actions):
    """actions int(u*A), returns U[-2,2) (test_nnet.cpp:43-55 style)."""
    u = uniforms(derive_seed(seed, [0x61637473]), 2 * B)
    actions = (u[:B] * n_actions).astype(np.int32)
    rets = u[B:] * 4.0 - 2.0
    return actions, rets
