"""DeviceLoop -- the device-resident GA3C iteration that bench.py times.

A step is one GA3C iteration for N_A agents on one GPU:
  t_max predictor batches   forward(N_A frames) + inverse-CDF sampling
                            (pipeline.cpp:65-93, util.hpp:46-54) on the
                            predictor-only parameter slot
  n-step returns            per agent segment (returns.cpp:8-26),
                            bootstrapped with the value just played
  trainer updates           N_A*t_max / min_train_batch updates, each
                            loss_and_gradients + RMSProp (pipeline.cpp:241-306)

N_T trainers in flight (GA3C's trainer threads): update U's gradient runs on
trainer context U % N_T (own stream and workspace) against parameter version
max(0, U - N_T + 1); the RMSProp steps stay serialized in update order on the
main stream and write out of place into a ring of R >= N_T + 1 slots, so a
trainer never reads a version being overwritten (slot = version mod R).  With
overlap, the predictor phase of step i runs beside the trainers of step i,
which consume step i-1's experiences (the training queue decouples them), and
the predictor reads a slot the trainers never write, refreshed with the
step's last version at the end of the step.

This module is shared by bench.py (timing) and tests/test_loop_parity_gpu.py
(the oracle replays exactly this schedule), so the parity test checks the
code path the benchmark measures.

Policy lag in the reference's own metric (pipeline.cpp:289-291,
applied_on - produced_version): experiences of step i are produced at the
version published at the end of step i-1, i.e. ``updates * i``; they are
applied by updates U = updates * (i + 1) + u on top of version U, so the lag
is updates + u and its mean over a step is ``updates + (updates - 1) / 2``
(23.5 for 16 updates per step).  Without overlap the predictor runs first in
the step on the step's starting version and the trainers consume that step's
experiences: the lag is u, mean (updates - 1) / 2.
"""
from __future__ import annotations

FRAME = (84, 84, 4)
FRAME_BYTES = 84 * 84 * 4
GMAX = 8  # steps one CUDA graph may chain


def ring_size(NT: int, updates: int) -> int:
    """Smallest R >= N_T + 1 dividing the updates per step (every step then
    starts from ring slot 0, so one graph per input set replays any step)."""
    sizes = [r for r in range(NT + 1, updates + 1) if updates % r == 0]
    if not sizes:
        raise ValueError("N_T must be below the updates per step")
    return sizes[0]


def grad_version(U: int, NT: int) -> int:
    """Parameter version update U's gradient is computed on."""
    return max(0, U - NT + 1)


def mean_policy_lag(updates: int, overlap: bool) -> float:
    """Mean applied_on - produced_version (pipeline.cpp:289-291) of the device step."""
    return updates + (updates - 1) / 2 if overlap else (updates - 1) / 2


class DeviceLoop:
    """The schedule above over the C ABI.  Inputs are device tensors:
    frames u8 [sets, N_A, t_max, 84, 84, 4]; uni f64 [sets, t_max, N_A];
    rewards f64 [sets, N_A, t_max]; terminal u8 [sets, N_A]."""

    def __init__(self, model, ctx, NA, T, TB, NT, frames, uni, rewards, terminal, *, trainer_sms=0,
                 pred_sms=0, overlap=True, world=1, device="cuda", hyper=None, dp_update=None):
        import torch

        from . import _abi, dp
        self.torch, self._abi, self.dp = torch, _abi, dp
        self.model, self.ctx = model, ctx
        self.NA, self.T, self.TB, self.NT = NA, T, TB, NT
        self.n = NA * T
        self.updates = self.n // TB
        if self.n % TB or TB % T:
            raise ValueError("train batch must cover whole agent segments")
        self.frames, self.uni, self.rewards, self.terminal = frames, uni, rewards, terminal
        self.sets = frames.shape[0]
        self.world = world
        self.hyper = hyper or _abi.default_hyper()
        if self.hyper.grad_clip_norm != 0.0 and NT > 1:
            raise ValueError("clipping with several trainers in flight is not wired here")
        self.stream = torch.cuda.ExternalStream(ctx.stream)
        self.P = model.P
        self.offsets = torch.arange(0, self.n + 1, T, dtype=torch.int32, device=device)
        # double-buffered experience (actions, n-step returns)
        self.actions2 = torch.zeros((2, NA, T), dtype=torch.int32, device=device)
        self.rets2 = torch.zeros((2, NA, T), dtype=torch.float64, device=device)
        self.fstride = T * FRAME_BYTES
        self.overlap = NT > 1 and overlap
        self.grad_view = dp.grad_view(ctx, self.P, device) if world > 1 else None
        self.dp_update = dp_update  # data-parallel exchange for NT > 1 (fused kernel or NCCL), or None
        self.nccl = None  # dp.NcclComm for the NCCL exchange (dp.nccl_update, and NT == 1)
        if NT > 1:
            self.R = ring_size(NT, self.updates)
            self.ring = model.ring(self.R + 1)  # + the predictor's slot, never written by a trainer
            self.pred_slot = self.ring[self.R]
            self.tctx = [_abi.Context(model, TB) for _ in range(NT)]
            self.tstream = [torch.cuda.ExternalStream(c.stream) for c in self.tctx]
            self.tgrad = [dp.grad_view(c, self.P, device) for c in self.tctx] if world > 1 else None
            n_ev = self.updates * GMAX
            self.ev_g = [torch.cuda.Event() for _ in range(n_ev)]
            self.ev_a = [torch.cuda.Event() for _ in range(n_ev)]
            self.ev_r = torch.cuda.Event()
            self.ev_p = [torch.cuda.Event() for _ in range(GMAX)]
            self.ev_end = [torch.cuda.Event() for _ in range(GMAX)]
            for c in self.tctx:
                c.set_sm_budget(trainer_sms)
        else:
            self.R, self.ring, self.tctx = 1, None, []
            self.slot, _ = model.acquire()
        self.pctx = _abi.Context(model, NA) if self.overlap else ctx
        if self.overlap:
            self.pctx.set_sm_budget(pred_sms)
        self.pstream = torch.cuda.ExternalStream(self.pctx.stream) if self.overlap else self.stream
        self.lv = self.pctx.last_values_ptr()
        self.contexts = [ctx] + (self.tctx if NT > 1 else []) + ([self.pctx] if self.overlap else [])

    # ------------------------------------------------------------ phases
    def predict(self, i, b):
        """t_max predictor batches of N_A agents, sampling, n-step returns -> buffer b."""
        s = i % self.sets
        fr = self.frames[s].data_ptr()
        pslot = self.pred_slot if self.NT > 1 else self.slot
        acts, rts = self.actions2[b], self.rets2[b]
        for t in range(self.T):
            self.pctx.forward_dev(fr + t * FRAME_BYTES, self.NA, True, slot=pslot, stride=self.fstride)
            self.pctx.sample_dev(self.uni[s, t].data_ptr(), self.NA, acts.data_ptr() + 4 * t, stride=self.T)
        self.pctx.compute_returns_dev(self.rewards[s].data_ptr(), self.offsets.data_ptr(), self.NA,
                                      self.terminal[s].data_ptr(), self.lv, self.hyper.gamma, rts.data_ptr())

    def step(self, i, pos=0):
        """One GA3C iteration.  pos = position inside a multi-step graph (0 =
        first, or eager): the update index U = pos * updates + u is continuous
        across chained steps, so trainer U waits only for apply U - N_T."""
        TB, NT = self.TB, self.NT
        if NT == 1:
            self.predict(i, 0)
            fr = self.frames[i % self.sets].data_ptr()
            for u in range(self.updates):
                self.dp.dp_update(self.ctx, fr + u * TB * FRAME_BYTES, True, self.actions2[0].data_ptr() + 4 * u * TB,
                                  self.rets2[0].data_ptr() + 8 * u * TB, TB, self.slot, self.grad_view, self.stream,
                                  self.world, self.nccl)
            return
        base = pos * self.updates
        stream, tstream = self.stream, self.tstream
        if self.overlap:
            if pos == 0:
                self.ev_r.record(stream)
                self.ev_r.wait(self.pstream)
            else:
                self.ev_end[pos - 1].wait(self.pstream)
            self.predict(i, i % 2)
            self.ev_p[pos].record(self.pstream)
            ti, b = i - 1, (i - 1) % 2
            ready = self.ev_r if pos == 0 else self.ev_p[pos - 1]  # this step's experiences exist
        else:
            self.predict(i, 0)
            self.ev_r.record(stream)
            ti, b = i, 0
            ready = self.ev_r
        fr = self.frames[ti % self.sets].data_ptr()
        acts, rts = self.actions2[b], self.rets2[b]
        R, ring = self.R, self.ring
        for u in range(self.updates):
            U = base + u
            j = U % NT
            if u < NT:
                ready.wait(tstream[j])
            if U >= NT:
                self.ev_a[U - NT].wait(tstream[j])  # version U - N_T + 1 exists; context j's last gradient was applied
            self.tctx[j].loss_grad_dev(fr + u * TB * FRAME_BYTES, True, acts.data_ptr() + 4 * u * TB,
                                       rts.data_ptr() + 8 * u * TB, TB, ring[(U - NT + 1) % R],
                                       apply_clip=self.world == 1)
            self.ev_g[U].record(tstream[j])
            self.ev_g[U].wait(stream)
            if self.dp_update is not None:
                self.dp_update(self, j, U)
            else:
                self.ctx.apply_slots_dev(self.tctx[j], ring[U % R], ring[(U + 1) % R])
            self.ev_a[U].record(stream)
        if self.overlap:
            self.ev_p[pos].wait(stream)  # the predictor is done reading its slot
        self.ctx.copy_slot_dev(ring[self.updates % R], self.pred_slot)
        self.ev_end[pos].record(stream)

    # ---------------------------------------------------------- graphs
    def capture(self, G, first=0):
        """One CUDA graph per input set, each chaining G steps (positions
        0..G-1, update index continuous).  Returns (graphs, launches per step)."""
        graphs = []
        l0 = self.launches()
        for s in range(self.sets):
            self.ctx.graph_begin()
            for pos in range(G):
                self.step(first + s * G + pos, pos)
            graphs.append(self.ctx.graph_end())
        return graphs, (self.launches() - l0) // (self.sets * G)

    def launch(self, gid):
        self.ctx.graph_launch(gid)

    # ------------------------------------------------------- probes
    def time_kernel(self, tag, li=-1):
        for c in self.contexts:
            c.time_kernel(tag, li)

    def kernel_time(self):
        ms = cnt = 0
        for c in self.contexts:
            a, b = c.kernel_time()
            ms, cnt = ms + a, cnt + b
        return ms, cnt

    def launches(self):
        return sum(c.launches() for c in self.contexts)

    def latest_slot(self):
        """Ring slot holding the newest version after whole steps (slot = version mod R)."""
        return self.ring[0] if self.NT > 1 else self.slot

    def sync(self):
        for c in self.contexts:
            c.sync()
