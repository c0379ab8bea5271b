"""Data-parallel trainer step: one process per GPU.

The reference's loss_and_gradients returns the SUMMED gradient over its batch
(nnet.hpp:88-94), so splitting a merged training batch across G
replicas and summing the per-replica gradients with one NCCL all-reduce gives
the single-device gradient of the whole batch (up to fp32 summation order).
The optional global-norm clip (nnet.cpp:281-289) must then run on the reduced
gradient, and every replica applies the same RMSProp step to the same
parameters, so replicas stay bit-identical and their versions advance
together.  Predictors are sharded per GPU by agent (agent_id mod G); they
need no exchange.

The functions here are the host-side plumbing; the arithmetic is the C ABI's
(ga3c_loss_grad_dev with apply_clip=0, ga3c_clip_grad, ga3c_apply_rmsprop_dev)
and the reduction is torch.distributed (NCCL on the B200 box, gloo in the
CPU tests).
"""
from __future__ import annotations


def shard(n: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of n items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def agents_of(rank: int, world: int, n_agents: int):
    """Predictor sharding: agent ids served by this GPU (agent_id mod G)."""
    return [a for a in range(n_agents) if a % world == rank]


def grad_view(ctx, P: int, device):
    """Zero-copy torch view of a context's device gradient buffer."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (P,), "typestr": "<f4", "data": (ctx.grad_ptr(), False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_View(), device=device)


def allreduce_sum_(t, stream=None):
    """In-place sum over the default process group, ordered on `stream`."""
    import torch
    import torch.distributed as dist
    if stream is None:
        dist.all_reduce(t)
        return t
    with torch.cuda.stream(stream):
        dist.all_reduce(t)
    return t


def dp_update(ctx, d_states, u8, d_actions, d_returns, B_local, slot, gview, stream, world):
    """One data-parallel update on this rank's shard: local summed gradient,
    all-reduce(sum), clip on the reduced gradient, identical RMSProp."""
    ctx.loss_grad_dev(d_states, u8, d_actions, d_returns, B_local, slot, apply_clip=world == 1)
    if world > 1:
        allreduce_sum_(gview, stream)
        ctx.clip_grad()
    ctx.apply_rmsprop_dev()
