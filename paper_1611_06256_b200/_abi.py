"""ctypes binding of the C ABI in include/ga3c.h (libga3c_b200.so).

This is the Python side of the drop-in boundary: the same entry points a
maintainer would bind from the reference's pybind11 module
(proj/bindings/qac_module.cpp) -- see INTEGRATION.md.  There is no CPU path:
if the shared library is missing this module raises ImportError, and every
compute call raises RuntimeError when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libga3c_b200.so")

MAX_CONV = 4
MAX_HIDDEN = 4

OK = 0
INVALID_ARGUMENT = 1
NONFINITE_INPUT = 2
CUDA_ERROR = 3
NCCL_ERROR = 4
NOT_APPLIED = 5
OUT_OF_MEMORY = 6


class NetSpec(C.Structure):
    """ga3c_net_spec (include/ga3c.h)."""

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


class HyperC(C.Structure):
    """ga3c_hyper (include/ga3c.h) = Hyperparams nnet.hpp:20-31."""

    _fields_ = [
        ("gamma", C.c_double), ("t_max", C.c_int), ("beta", C.c_double),
        ("eps_log", C.c_double), ("eta", C.c_double), ("alpha", C.c_double),
        ("eps_rms", C.c_double), ("value_loss_weight", C.c_double),
        ("grad_clip_norm", C.c_double), ("clip_rewards", C.c_int),
    ]


class PipelineOpts(C.Structure):
    """ga3c_pipeline_opts (include/ga3c.h)."""

    _fields_ = [
        ("net", NetSpec), ("hyper", HyperC),
        ("env_kind", C.c_int), ("n_contexts", C.c_int), ("env_actions", C.c_int), ("grid_size", C.c_int),
        ("step_delay_us", C.c_longlong), ("episode_len", C.c_int), ("action_repeat", C.c_int),
        ("n_agents", C.c_int), ("n_predictors", C.c_int), ("n_trainers", C.c_int),
        ("pred_batch_max", C.c_int), ("min_train_batch", C.c_int), ("train_queue_cap", C.c_int),
        ("pred_queue_cap", C.c_int),
        ("max_updates", C.c_longlong), ("max_seconds", C.c_double), ("target_score", C.c_double),
        ("has_target_score", C.c_int),
        ("seed", C.c_ulonglong), ("anneal", C.c_int), ("anneal_batches", C.c_int), ("epoch_s", C.c_double),
        ("max_agents", C.c_int), ("max_predictors", C.c_int), ("max_trainers", C.c_int),
        ("metrics_interval_s", C.c_double),
        ("greedy", C.c_int), ("sync_after_submit", C.c_int), ("capture_trajectory", C.c_int), ("device", C.c_int),
        ("device_frames", C.c_int), ("trainer_sms", C.c_int), ("predictor_sms", C.c_int),
    ]


class RunReportC(C.Structure):
    """ga3c_run_report (include/ga3c.h)."""

    _fields_ = [
        ("total_updates", C.c_longlong), ("skipped_updates", C.c_longlong),
        ("total_predictions", C.c_longlong), ("total_episodes", C.c_longlong),
        ("wall_time_s", C.c_double), ("avg_tps", C.c_double), ("avg_pps", C.c_double),
        ("avg_samples_per_s", C.c_double), ("mean_lag", C.c_double), ("final_rolling_score", C.c_double),
        ("experiences_produced", C.c_longlong), ("experiences_trained", C.c_longlong),
        ("experiences_dropped", C.c_longlong), ("experiences_left_queued", C.c_longlong),
        ("final_n_agents", C.c_int), ("final_n_predictors", C.c_int), ("final_n_trainers", C.c_int),
        ("final_pred_batch_max", C.c_int), ("final_min_train_batch", C.c_int),
        ("final_version", C.c_ulonglong),
        ("n_trajectory", C.c_int), ("n_anneal", C.c_int), ("n_frames", C.c_int),
        ("last_frame_tps", C.c_double), ("last_frame_pps", C.c_double), ("last_frame_pred_batch_mean", C.c_double),
    ]


class AnnealEntry(C.Structure):
    _fields_ = [("n_agents", C.c_int), ("n_predictors", C.c_int), ("n_trainers", C.c_int),
                ("pred_batch_max", C.c_int), ("min_train_batch", C.c_int), ("measured_tps", C.c_double),
                ("accepted", C.c_int)]


_P = C.c_void_p
_SIGS = {
    "ga3c_status_string": (C.c_char_p, [C.c_int]),
    "ga3c_default_hyper": (None, [C.POINTER(HyperC)]),
    "ga3c_validate_spec": (C.c_int, [C.POINTER(NetSpec)]),
    "ga3c_validate_hyper": (C.c_int, [C.POINTER(HyperC)]),
    "ga3c_param_count": (C.c_size_t, [C.POINTER(NetSpec)]),
    "ga3c_input_dim": (C.c_size_t, [C.POINTER(NetSpec)]),
    "ga3c_init_params": (C.c_int, [C.POINTER(NetSpec), C.c_uint64, _P, _P]),
    "ga3c_model_create": (_P, [C.POINTER(NetSpec), C.POINTER(HyperC), C.c_int, C.POINTER(C.c_int)]),
    "ga3c_model_destroy": (None, [_P]),
    "ga3c_model_load": (C.c_int, [_P, _P, _P, C.c_uint64]),
    "ga3c_model_read": (C.c_int, [_P, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_model_version": (C.c_uint64, [_P]),
    "ga3c_model_param_count": (C.c_size_t, [_P]),
    "ga3c_model_n_actions": (C.c_int, [_P]),
    "ga3c_snapshot_acquire": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    "ga3c_snapshot_release": (C.c_int, [_P, C.c_int]),
    "ga3c_model_last_error": (C.c_char_p, [_P]),
    "ga3c_ctx_create": (_P, [_P, C.c_int, C.POINTER(C.c_int)]),
    "ga3c_ctx_destroy": (None, [_P]),
    "ga3c_ctx_stream": (_P, [_P]),
    "ga3c_ctx_sync": (C.c_int, [_P]),
    "ga3c_ctx_launches": (C.c_uint64, [_P]),
    "ga3c_forward_u8": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_forward_f32": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_forward64_u8": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_forward64_f32": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_forward_dev": (C.c_int, [_P, C.c_int, _P, C.c_int, C.c_longlong, C.c_int, _P, _P]),
    "ga3c_loss_grad_u8": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_int, _P, _P]),
    "ga3c_loss_grad_f32": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_int, _P, _P]),
    "ga3c_loss_grad_dev": (C.c_int, [_P, C.c_int, _P, C.c_int, C.c_longlong, _P, _P, C.c_int, C.c_int]),
    "ga3c_loss_grad_segments_u8": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, _P, C.c_int, _P, _P,
                                             C.c_double, C.c_int, _P, _P]),
    "ga3c_loss_grad_segments_f32": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, _P, _P, C.c_int, _P, _P,
                                              C.c_double, C.c_int, _P, _P]),
    "ga3c_ctx_grad": (_P, [_P]),
    "ga3c_ctx_last_values": (_P, [_P]),
    "ga3c_ctx_read_grad": (C.c_int, [_P, _P, _P]),
    "ga3c_clip_grad": (C.c_int, [_P]),
    "ga3c_check_grad": (C.c_int, [_P, _P]),
    "ga3c_allreduce_grads": (C.c_int, [_P, _P, _P]),
    "ga3c_nccl_unique_id": (C.c_int, [_P]),
    "ga3c_nccl_comm_init": (C.c_int, [C.c_int, _P, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ga3c_nccl_comm_destroy": (C.c_int, [_P]),
    "ga3c_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "ga3c_ctx_model": (_P, [_P]),
    "ga3c_model_read_slot": (C.c_int, [_P, C.c_int, _P, _P]),
    "ga3c_rmsprop_flat": (C.c_int, [C.POINTER(HyperC), C.c_int, C.c_size_t, _P, _P, _P, C.POINTER(C.c_int)]),
    "ga3c_apply_rmsprop": (C.c_int, [_P, _P, C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    "ga3c_apply_rmsprop_dev": (C.c_int, [_P]),
    "ga3c_ctx_read_dev_version": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "ga3c_compute_returns": (C.c_int, [_P, _P, _P, C.c_int, _P, _P, C.c_double, _P]),
    "ga3c_compute_returns_dev": (C.c_int, [_P, _P, _P, C.c_int, _P, _P, C.c_double, _P]),
    "ga3c_sample_actions_dev": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P, C.c_int]),
    "ga3c_ctx_time_kernel": (C.c_int, [_P, C.c_int, C.c_int]),
    "ga3c_default_pipeline_opts": (None, [C.POINTER(PipelineOpts)]),
    "ga3c_pipeline_run": (C.c_int, [C.POINTER(PipelineOpts), C.c_int, C.POINTER(RunReportC), _P, _P, C.c_int,
                                    _P, C.c_int, _P, C.c_int, C.c_char_p, C.c_int]),
    "ga3c_ctx_graph_begin": (C.c_int, [_P]),
    "ga3c_ctx_graph_end": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "ga3c_ctx_graph_launch": (C.c_int, [_P, C.c_int]),
    "ga3c_ctx_kernel_time": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "ga3c_ctx_timeline": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P, C.POINTER(C.c_int)]),
    "ga3c_model_ring": (C.c_int, [_P, C.c_int, _P]),
    "ga3c_apply_rmsprop_slots_dev": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "ga3c_copy_slot_dev": (C.c_int, [_P, C.c_int, C.c_int]),
    "ga3c_ctx_set_sm_budget": (C.c_int, [_P, C.c_int]),
    "ga3c_ctx_set_priority": (C.c_int, [_P, C.c_int]),
    "ga3c_frames_create": (_P, [_P, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "ga3c_frames_destroy": (None, [_P]),
    "ga3c_host_alloc": (_P, [C.c_size_t, C.POINTER(C.c_int)]),
    "ga3c_predict_frames64_async": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int, _P]),
    "ga3c_predict_collect64": (C.c_int, [_P, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_predict_frames_act64_async": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int, _P, _P]),
    "ga3c_predict_collect_act64": (C.c_int, [_P, _P, _P, _P, C.POINTER(C.c_uint64)]),
    "ga3c_host_free": (None, [_P]),
    "ga3c_trainer_pool_create": (_P, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "ga3c_trainer_pool_submit": (C.c_int, [_P, _P, _P, C.c_int, _P, _P, _P, C.c_int, _P, _P, C.c_double]),
    "ga3c_trainer_pool_submit_many": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_double]),
    "ga3c_trainer_pool_wait": (C.c_int, [_P, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "ga3c_trainer_pool_error": (C.c_char_p, [_P]),
    "ga3c_trainer_pool_destroy": (None, [_P]),
    "ga3c_predict_frames": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int, _P, _P, _P,
                                      C.POINTER(C.c_uint64)]),
    "ga3c_predict_frames64": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int, _P, _P, _P,
                                        C.POINTER(C.c_uint64)]),
    "ga3c_train_frames": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, _P, _P, _P, C.c_int, _P, _P, C.c_double,
                                    C.c_int, _P, _P]),
    "ga3c_frames_read": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "ga3c_dp_create": (_P, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "ga3c_dp_destroy": (None, [_P]),
    "ga3c_dp_signal": (_P, [_P]),
    "ga3c_dp_check": (C.c_int, [_P]),
    "ga3c_model_slot_theta": (C.c_int, [_P, C.c_int, C.POINTER(C.c_void_p)]),
    "ga3c_dp_apply": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P, _P, _P]),
    "ga3c_ipc_get_handle": (C.c_int, [_P, _P]),
    "ga3c_ipc_open_handle": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "ga3c_ipc_close": (C.c_int, [_P]),
}

K_TAGS = {"none": 0, "conv_fwd": 1, "fc_fwd": 2, "heads": 3, "loss_bwd": 4, "wgrad": 5, "dgrad": 6,
          "splitk": 7, "rmsprop": 8, "returns": 9, "sample": 10, "other": 11, "all": 12}

EXPORTED = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the GA3C hot path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class GA3CError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{lib.ga3c_status_string(status).decode()}: {msg}")


class InvalidArgument(GA3CError, ValueError):
    """Where the reference throws std::invalid_argument (pybind -> ValueError)."""


def check(status, msg=""):
    if status == OK:
        return
    if status in (INVALID_ARGUMENT, NONFINITE_INPUT):
        raise InvalidArgument(status, msg)
    raise GA3CError(status, msg)


def ptr(a):
    """Device/host pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def default_hyper():
    h = HyperC()
    lib.ga3c_default_hyper(C.byref(h))
    return h


class Model:
    """ga3c_model: device parameters + rms state, versioned snapshots."""

    def __init__(self, spec: NetSpec, hyper: HyperC, device: int = 0):
        st = C.c_int(0)
        self.spec, self.hyper = spec, hyper
        self.h = lib.ga3c_model_create(C.byref(spec), C.byref(hyper), device, C.byref(st))
        if not self.h:
            check(st.value, lib.ga3c_model_last_error(None).decode())
        self.P = int(lib.ga3c_model_param_count(self.h))
        self.device = device
        self.n_actions = spec.n_actions
        self.input_dim = int(spec.in_h) * int(spec.in_w) * int(spec.in_c)

    def close(self):
        if getattr(self, "h", None):
            lib.ga3c_model_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def error(self):
        return lib.ga3c_model_last_error(self.h).decode()

    def load(self, theta, g=None, version=0):
        theta = np.ascontiguousarray(theta, np.float32)
        g = None if g is None else np.ascontiguousarray(g, np.float32)
        assert theta.size == self.P
        check(lib.ga3c_model_load(self.h, ptr(theta), ptr(g), version), self.error())

    def read(self):
        th = np.zeros(self.P, np.float32)
        g = np.zeros(self.P, np.float32)
        v = C.c_uint64(0)
        check(lib.ga3c_model_read(self.h, ptr(th), ptr(g), C.byref(v)), self.error())
        return th, g, v.value

    def read_slot(self, slot):
        """theta and g of one parameter slot (after all in-flight writes)."""
        th = np.zeros(self.P, np.float32)
        g = np.zeros(self.P, np.float32)
        check(lib.ga3c_model_read_slot(self.h, slot, ptr(th), ptr(g)), self.error())
        return th, g

    def version(self):
        return int(lib.ga3c_model_version(self.h))

    def ring(self, n):
        """n caller-owned device slots for a multi-trainer device loop."""
        import numpy as np
        out = np.zeros(n, np.int32)
        check(lib.ga3c_model_ring(self.h, n, out.ctypes.data), self.error())
        return [int(x) for x in out]

    def acquire(self):
        s, v = C.c_int(0), C.c_uint64(0)
        check(lib.ga3c_snapshot_acquire(self.h, C.byref(s), C.byref(v)))
        return s.value, v.value

    def release(self, slot):
        check(lib.ga3c_snapshot_release(self.h, slot))


class Context:
    """ga3c_ctx: one CUDA stream + workspace for batches up to max_batch."""

    def __init__(self, model: Model, max_batch: int):
        st = C.c_int(0)
        self.model = model
        self.h = lib.ga3c_ctx_create(model.h, max_batch, C.byref(st))
        if not self.h:
            check(st.value, lib.ga3c_model_last_error(model.h).decode())
        self.max_batch = max_batch
        self.A = model.spec.n_actions

    def close(self):
        if getattr(self, "h", None):
            lib.ga3c_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    @property
    def stream(self):
        return lib.ga3c_ctx_stream(self.h)

    def sync(self):
        check(lib.ga3c_ctx_sync(self.h), self.model.error())

    def launches(self):
        return int(lib.ga3c_ctx_launches(self.h))

    # --- host-buffer calls (blocking) -------------------------------------
    def forward(self, states, slot=-1, fp64=False):
        """states: (B, H*W*C) or (B,H,W,C) uint8 frames or float32 states.
        fp64: pi as the device's fp64 softmax, V widened (ga3c_forward64_*)."""
        states = np.ascontiguousarray(states)
        B = states.shape[0]
        dt = np.float64 if fp64 else np.float32
        pi = np.zeros((B, self.A), dt)
        v = np.zeros(B, dt)
        ver = C.c_uint64(0)
        if states.dtype == np.uint8:
            fn = lib.ga3c_forward64_u8 if fp64 else lib.ga3c_forward_u8
            rc = fn(self.h, slot, ptr(states), B, ptr(pi), ptr(v), C.byref(ver))
        else:
            states = np.ascontiguousarray(states, np.float32)
            fn = lib.ga3c_forward64_f32 if fp64 else lib.ga3c_forward_f32
            rc = fn(self.h, slot, ptr(states), B, ptr(pi), ptr(v), C.byref(ver))
        check(rc, self.model.error())
        return pi, v, ver.value

    def loss_grad(self, states, actions, returns, slot=-1, apply_clip=True, want_grad=True):
        states = np.ascontiguousarray(states)
        B = states.shape[0]
        actions = np.ascontiguousarray(actions, np.int32)
        returns = np.ascontiguousarray(returns, np.float64)
        if actions.size != B or returns.size != B:
            raise InvalidArgument(INVALID_ARGUMENT, "returns/experiences length mismatch")
        d = np.zeros(self.model.P, np.float32) if want_grad else None
        sc = np.zeros(3, np.float64)
        if states.dtype == np.uint8:
            rc = lib.ga3c_loss_grad_u8(self.h, slot, ptr(states), ptr(actions), ptr(returns), B,
                                       int(apply_clip), ptr(d), ptr(sc))
        else:
            states = np.ascontiguousarray(states, np.float32)
            rc = lib.ga3c_loss_grad_f32(self.h, slot, ptr(states), ptr(actions), ptr(returns), B,
                                        int(apply_clip), ptr(d), ptr(sc))
        check(rc, self.model.error())
        return d, sc

    def loss_grad_segments(self, states, actions, rewards, seg_offsets, terminal, bootstrap, gamma,
                           slot=-1, apply_clip=True):
        """Trainer step with device-side n-step returns -> (scalars, returns)."""
        states = np.ascontiguousarray(states)
        B = states.shape[0]
        a = np.ascontiguousarray(actions, np.int32)
        r = np.ascontiguousarray(rewards, np.float64)
        off = np.ascontiguousarray(seg_offsets, np.int32)
        term = np.ascontiguousarray(terminal, np.uint8)
        boot = np.ascontiguousarray(bootstrap, np.float64)
        sc = np.zeros(3, np.float64)
        rets = np.zeros(B, np.float64)
        f = lib.ga3c_loss_grad_segments_u8 if states.dtype == np.uint8 else lib.ga3c_loss_grad_segments_f32
        if states.dtype != np.uint8:
            states = np.ascontiguousarray(states, np.float32)
        check(f(self.h, slot, ptr(states), B, ptr(a), ptr(r), ptr(off), len(off) - 1, ptr(term), ptr(boot),
                float(gamma), int(apply_clip), ptr(sc), ptr(rets)), self.model.error())
        return sc, rets

    def apply_rmsprop(self, dtheta=None):
        """SharedModel::apply -> (applied, applied_on_version)."""
        d = None if dtheta is None else np.ascontiguousarray(dtheta, np.float32)
        ap, on = C.c_int(0), C.c_uint64(0)
        rc = lib.ga3c_apply_rmsprop(self.h, ptr(d), C.byref(ap), C.byref(on))
        if rc == NOT_APPLIED:
            return False, None
        check(rc, self.model.error())
        return bool(ap.value), on.value

    def compute_returns(self, rewards, seg_offsets, terminal, bootstrap, gamma):
        r = np.ascontiguousarray(rewards, np.float64)
        off = np.ascontiguousarray(seg_offsets, np.int32)
        term = np.ascontiguousarray(terminal, np.uint8)
        boot = np.ascontiguousarray(bootstrap, np.float64)
        out = np.zeros(r.size, np.float64)
        check(lib.ga3c_compute_returns(self.h, ptr(r), ptr(off), len(off) - 1, ptr(term), ptr(boot),
                                       float(gamma), ptr(out)), self.model.error())
        return out

    def read_grad(self):
        d = np.zeros(self.model.P, np.float32)
        sc = np.zeros(3, np.float64)
        check(lib.ga3c_ctx_read_grad(self.h, ptr(d), ptr(sc)), self.model.error())
        return d, sc

    # --- device-resident calls (async on self.stream) ----------------------
    def forward_dev(self, d_states, B, u8, d_pi=None, d_v=None, slot=None, stride=0):
        s = self.model.acquire()[0] if slot is None else slot
        rc = lib.ga3c_forward_dev(self.h, s, d_states, int(u8), stride, B, d_pi, d_v)
        if slot is None:
            self.model.release(s)  # caller owns ordering (single-threaded device loop)
        check(rc, self.model.error())

    def loss_grad_dev(self, d_states, u8, d_actions, d_returns, B, slot, apply_clip=True, stride=0):
        check(lib.ga3c_loss_grad_dev(self.h, slot, d_states, int(u8), stride, d_actions, d_returns, B,
                                     int(apply_clip)), self.model.error())

    def apply_slots_dev(self, grad_from, src_slot, dst_slot):
        check(lib.ga3c_apply_rmsprop_slots_dev(self.h, grad_from.h if grad_from is not None else None, src_slot,
                                               dst_slot), self.model.error())

    def set_sm_budget(self, sms):
        check(lib.ga3c_ctx_set_sm_budget(self.h, sms), self.model.error())

    def set_priority(self, level):
        """ga3c_ctx_set_priority: 0 = highest (default), k = k levels lower."""
        check(lib.ga3c_ctx_set_priority(self.h, level), self.model.error())

    def copy_slot_dev(self, src_slot, dst_slot):
        check(lib.ga3c_copy_slot_dev(self.h, src_slot, dst_slot), self.model.error())

    def apply_rmsprop_dev(self):
        check(lib.ga3c_apply_rmsprop_dev(self.h), self.model.error())

    def compute_returns_dev(self, d_rew, d_off, n_seg, d_term, d_boot, gamma, d_out):
        check(lib.ga3c_compute_returns_dev(self.h, d_rew, d_off, n_seg, d_term, d_boot, float(gamma),
                                           d_out), self.model.error())

    def sample_dev(self, d_u, B, d_actions, d_pi=None, stride=1):
        check(lib.ga3c_sample_actions_dev(self.h, d_pi, d_u, B, self.A, d_actions, stride),
              self.model.error())

    def last_values_ptr(self):
        return lib.ga3c_ctx_last_values(self.h)

    def grad_ptr(self):
        return lib.ga3c_ctx_grad(self.h)

    def clip_grad(self):
        check(lib.ga3c_clip_grad(self.h), self.model.error())

    def check_grad(self, grad_from=None):
        """Recompute the non-finite flag of the (all-reduced) gradient of
        grad_from (default: this context), on this context's stream."""
        check(lib.ga3c_check_grad(self.h, grad_from.h if grad_from is not None else None), self.model.error())

    def time_kernel(self, tag, layer=-1):
        check(lib.ga3c_ctx_time_kernel(self.h, K_TAGS[tag] if isinstance(tag, str) else tag, layer))

    def kernel_time(self):
        """(total_ms, launches) of the probed kernel class since the last call."""
        ms, n = C.c_double(0), C.c_uint64(0)
        check(lib.ga3c_ctx_kernel_time(self.h, C.byref(ms), C.byref(n)), self.model.error())
        return ms.value, n.value

    def timeline(self, cap=4096):
        """Per-launch (tag, layer, stream, start_ms, end_ms) since the last read
        (after time_kernel("all"))."""
        import numpy as np
        st, en = np.zeros(cap), np.zeros(cap)
        tg, ly, sm = (np.zeros(cap, np.int32) for _ in range(3))
        n = C.c_int(0)
        check(lib.ga3c_ctx_timeline(self.h, cap, st.ctypes.data, en.ctypes.data, tg.ctypes.data, ly.ctypes.data,
                                    sm.ctypes.data, C.byref(n)), self.model.error())
        names = {v: k for k, v in K_TAGS.items()}
        return [(names.get(int(tg[i]), str(tg[i])), int(ly[i]), int(sm[i]), float(st[i]), float(en[i]))
                for i in range(n.value)]

    def graph_begin(self):
        check(lib.ga3c_ctx_graph_begin(self.h), self.model.error())

    def graph_end(self):
        gid = C.c_int(-1)
        check(lib.ga3c_ctx_graph_end(self.h, C.byref(gid)), self.model.error())
        return gid.value

    def graph_launch(self, gid):
        check(lib.ga3c_ctx_graph_launch(self.h, gid), self.model.error())

    def dev_version(self):
        v = C.c_uint64(0)
        check(lib.ga3c_ctx_read_dev_version(self.h, C.byref(v)), self.model.error())
        return v.value


class Frames:
    """Device frame-stack store (ga3c_frames_*): agents push their newest
    frame; stacked states stay on the device for prediction and training."""

    def __init__(self, model: Model, n_agents: int, history: int):
        st = C.c_int(0)
        self.h = lib.ga3c_frames_create(model.h, n_agents, history, C.byref(st))
        if not self.h:
            check(st.value or 3, model.error())
        self.model = model
        self.n_agents, self.history = n_agents, history

    def close(self):
        if getattr(self, "h", None):
            lib.ga3c_frames_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def read(self, agent: int, slot: int):
        import numpy as np
        out = np.empty(self.model.input_dim, np.uint8)
        check(lib.ga3c_frames_read(self.h, agent, slot, out.ctypes.data))
        return out


def predict_frames(ctx: "Context", frames: Frames, new_frames, agents, resets=None, slot=-1, fp64=False):
    """-> (pi [n][A], v [n], state_slots [n], version); fp64 = the device's
    fp64 softmax and V (ga3c_predict_frames64)."""
    import numpy as np
    nf = np.ascontiguousarray(new_frames, np.uint8)
    ag = np.ascontiguousarray(agents, np.int32)
    n = len(ag)
    rs = None if resets is None else np.ascontiguousarray(resets, np.uint8)
    dt = np.float64 if fp64 else np.float32
    pi = np.empty((n, ctx.model.n_actions), dt)
    v = np.empty(n, dt)
    slots = np.empty(n, np.int32)
    ver = C.c_uint64(0)
    fn = lib.ga3c_predict_frames64 if fp64 else lib.ga3c_predict_frames
    check(fn(ctx.h, slot, frames.h, nf.ctypes.data, ag.ctypes.data,
                                  None if rs is None else rs.ctypes.data, n, slots.ctypes.data, pi.ctypes.data,
                                  v.ctypes.data, C.byref(ver)), ctx.model.error())
    return pi, v, slots, ver.value


def predict_frames_async(ctx: "Context", frames: Frames, new_frames, agents, resets=None, slot=-1):
    """Enqueue a frame-store prediction (ga3c_predict_frames64_async) -> state_slots;
    predict_collect(ctx) returns (pi fp64 [n][A], v [n], version).  Keep
    new_frames alive and unchanged until collected."""
    import numpy as np
    nf = np.ascontiguousarray(new_frames, np.uint8)
    ag = np.ascontiguousarray(agents, np.int32)
    n = len(ag)
    rs = None if resets is None else np.ascontiguousarray(resets, np.uint8)
    slots = np.empty(n, np.int32)
    check(lib.ga3c_predict_frames64_async(ctx.h, slot, frames.h, nf.ctypes.data, ag.ctypes.data,
                                          None if rs is None else rs.ctypes.data, n, slots.ctypes.data),
          ctx.model.error())
    ctx._pending = (n, nf, ag, rs)  # the buffers stay referenced until collected
    return slots


def predict_collect(ctx: "Context"):
    import numpy as np
    n = ctx._pending[0]
    pi = np.empty((n, ctx.model.n_actions), np.float64)
    v = np.empty(n, np.float64)
    ver = C.c_uint64(0)
    check(lib.ga3c_predict_collect64(ctx.h, pi.ctypes.data, v.ctypes.data, C.byref(ver)), ctx.model.error())
    ctx._pending = None
    return pi, v, ver.value


def predict_frames_act_async(ctx: "Context", frames: Frames, new_frames, agents, u, resets=None, slot=-1,
                             slots=None):
    """Enqueue a frame-store prediction whose actions are drawn on the device
    from the agents' uniforms u (ga3c_predict_frames_act64_async) ->
    state_slots (into `slots` when given); predict_collect_act(ctx) returns
    (actions, v, pi or None, version)."""
    import numpy as np
    nf = np.ascontiguousarray(new_frames, np.uint8)
    ag = np.ascontiguousarray(agents, np.int32)
    uu = np.ascontiguousarray(u, np.float64)
    n = len(ag)
    if uu.shape[0] != n:
        raise InvalidArgument(INVALID_ARGUMENT, "one uniform per agent")
    rs = None if resets is None else np.ascontiguousarray(resets, np.uint8)
    if slots is None:
        slots = np.empty(n, np.int32)
    check(lib.ga3c_predict_frames_act64_async(ctx.h, slot, frames.h, nf.ctypes.data, ag.ctypes.data,
                                              None if rs is None else rs.ctypes.data, n, uu.ctypes.data,
                                              slots.ctypes.data), ctx.model.error())
    ctx._pending = (n, nf, ag, rs, uu)
    return slots


def predict_collect_act(ctx: "Context", actions=None, want_pi=False):
    import numpy as np
    n = ctx._pending[0]
    if actions is None:
        actions = np.empty(n, np.int32)
    v = np.empty(n, np.float64)
    pi = np.empty((n, ctx.model.n_actions), np.float64) if want_pi else None
    ver = C.c_uint64(0)
    check(lib.ga3c_predict_collect_act64(ctx.h, actions.ctypes.data, v.ctypes.data,
                                         None if pi is None else pi.ctypes.data, C.byref(ver)), ctx.model.error())
    ctx._pending = None
    return actions, v, pi, ver.value


def train_frames(ctx: "Context", frames: Frames, agents, state_slots, actions, rewards, seg_offsets, terminal,
                 bootstrap, gamma, apply_clip=True, slot=-1):
    """-> (scalars [3], returns [B])."""
    import numpy as np
    ag = np.ascontiguousarray(agents, np.int32)
    sl = np.ascontiguousarray(state_slots, np.int32)
    ac = np.ascontiguousarray(actions, np.int32)
    rw = np.ascontiguousarray(rewards, np.float64)
    off = np.ascontiguousarray(seg_offsets, np.int32)
    te = np.ascontiguousarray(terminal, np.uint8)
    bo = np.ascontiguousarray(bootstrap, np.float64)
    B = len(ag)
    sc = np.empty(3)
    rets = np.empty(B)
    check(lib.ga3c_train_frames(ctx.h, slot, frames.h, ag.ctypes.data, sl.ctypes.data, B, ac.ctypes.data,
                                rw.ctypes.data, off.ctypes.data, len(off) - 1, te.ctypes.data, bo.ctypes.data,
                                gamma, 1 if apply_clip else 0, sc.ctypes.data, rets.ctypes.data), ctx.model.error())
    return sc, rets


class TrainerPool:
    """Native TrainingQueue + trainer threads (ga3c_trainer_pool_*): submit()
    hands a segment batch to C++ trainers (train_frames + apply_rmsprop on
    their own contexts) and returns; wait() blocks until all are applied."""

    def __init__(self, model: Model, frames: Frames, n_threads: int, max_batch: int, sms: int = 0,
                 queue_cap: int = 16):
        st = C.c_int(0)
        self.h = lib.ga3c_trainer_pool_create(model.h, frames.h, n_threads, max_batch, sms, queue_cap,
                                              C.byref(st))
        if not self.h:
            check(st.value or 3, model.error())
        self.model = model

    def submit(self, agents, state_slots, actions, rewards, seg_offsets, terminal, bootstrap, gamma):
        import numpy as np
        ag = np.ascontiguousarray(agents, np.int32)
        sl = np.ascontiguousarray(state_slots, np.int32)
        ac = np.ascontiguousarray(actions, np.int32)
        rw = np.ascontiguousarray(rewards, np.float64)
        off = np.ascontiguousarray(seg_offsets, np.int32)
        te = np.ascontiguousarray(terminal, np.uint8)
        bo = np.ascontiguousarray(bootstrap, np.float64)
        check(lib.ga3c_trainer_pool_submit(self.h, ag.ctypes.data, sl.ctypes.data, len(ag), ac.ctypes.data,
                                           rw.ctypes.data, off.ctypes.data, len(off) - 1, te.ctypes.data,
                                           bo.ctypes.data, gamma), self.error())

    def submit_many(self, batch_off, seg_base, agents, state_slots, actions, rewards, seg_offsets, terminal,
                    bootstrap, gamma):
        """Several batches in one call (ga3c_trainer_pool_submit_many): batch i =
        samples [batch_off[i], batch_off[i+1]), segments [seg_base[i],
        seg_base[i+1]), its offsets at seg_offsets[seg_base[i] + i ...]."""
        import numpy as np
        arr = [np.ascontiguousarray(batch_off, np.int32), np.ascontiguousarray(seg_base, np.int32),
               np.ascontiguousarray(agents, np.int32), np.ascontiguousarray(state_slots, np.int32),
               np.ascontiguousarray(actions, np.int32), np.ascontiguousarray(rewards, np.float64),
               np.ascontiguousarray(seg_offsets, np.int32), np.ascontiguousarray(terminal, np.uint8),
               np.ascontiguousarray(bootstrap, np.float64)]
        check(lib.ga3c_trainer_pool_submit_many(self.h, len(arr[0]) - 1, *[a.ctypes.data for a in arr], gamma),
              self.error())

    def wait(self):
        """-> (updates applied, updates rejected) so far."""
        u, r = C.c_longlong(0), C.c_longlong(0)
        check(lib.ga3c_trainer_pool_wait(self.h, C.byref(u), C.byref(r)), self.error())
        return u.value, r.value

    def error(self):
        return (lib.ga3c_trainer_pool_error(self.h) or b"").decode() if self.h else ""

    def close(self):
        if getattr(self, "h", None):
            lib.ga3c_trainer_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class FusedDP:
    """ga3c_dp: the fused reduce-scatter + RMSProp + all-gather update of one
    rank (include/ga3c.h).  `peers` are per-rank pointer lists as mapped in
    this process (see dp.FusedAllreduce for the CUDA IPC exchange)."""

    def __init__(self, model: Model, rank: int, world: int, ctas: int = 32):
        st = C.c_int(0)
        self.model = model
        self.rank, self.world = rank, world
        self.h = lib.ga3c_dp_create(model.h, rank, world, ctas, C.byref(st))
        if not self.h:
            check(st.value, model.error())

    def close(self):
        if getattr(self, "h", None):
            lib.ga3c_dp_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def signal_ptr(self):
        return lib.ga3c_dp_signal(self.h)

    def check(self):
        check(lib.ga3c_dp_check(self.h), self.model.error())

    def apply(self, ctx, grad_from, src_slot, dst_slot, grads, theta_dst, signals):
        W = self.world
        arr = lambda xs: (C.c_void_p * W)(*[C.c_void_p(int(x)) for x in xs])
        check(lib.ga3c_dp_apply(ctx.h, self.h, grad_from.h if grad_from is not None else None, src_slot, dst_slot,
                                arr(grads), arr(theta_dst), arr(signals)), self.model.error())


def slot_theta_ptr(model: Model, slot: int) -> int:
    p = C.c_void_p(0)
    check(lib.ga3c_model_slot_theta(model.h, slot, C.byref(p)), model.error())
    return int(p.value)


def ipc_handle(dev_ptr: int) -> bytes:
    buf = (C.c_char * 64)()
    check(lib.ga3c_ipc_get_handle(C.c_void_p(dev_ptr), buf))
    return bytes(buf)


def ipc_open(handle: bytes) -> int:
    p = C.c_void_p(0)
    buf = (C.c_char * 64).from_buffer_copy(handle)
    check(lib.ga3c_ipc_open_handle(buf, C.byref(p)))
    return int(p.value)
