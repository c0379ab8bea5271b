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
CPU tests).  FusedUpdate replaces all-reduce + RMSProp with one kernel per
update over NVLink peer memory (ga3c_dp_apply: reduce-scatter, sharded
RMSProp, all-gather of theta'), wiring the peers' buffers with CUDA IPC.
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


def dp_update(ctx, d_states, u8, d_actions, d_returns, B_local, slot, gview, stream, world, comm=None):
    """One data-parallel update on this rank's shard: local summed gradient,
    all-reduce(sum) (the library's NCCL entry when `comm` is a NcclComm, else
    torch.distributed), clip on the reduced gradient, identical RMSProp."""
    ctx.loss_grad_dev(d_states, u8, d_actions, d_returns, B_local, slot, apply_clip=world == 1)
    if world > 1 and comm is not None:
        comm.allreduce(ctx)
        ctx.clip_grad()
    elif world > 1:
        allreduce_sum_(gview, stream)
        # the reject decision must see the SUMMED gradient on every rank
        # (nnet.cpp:299-301): a rank whose own shard was finite would
        # otherwise apply a non-finite sum the others reject
        ctx.check_grad()
        ctx.clip_grad()
    ctx.apply_rmsprop_dev()


class NcclComm:
    """An NCCL communicator of the library's own entry points
    (ga3c_nccl_comm_init / ga3c_allreduce_grads): rank 0
    draws the id and the torch process group broadcasts it."""

    def __init__(self, rank, world, device):
        import ctypes as C

        from . import _abi
        self._abi = _abi
        uid = (C.c_char * 128)()
        if rank == 0:
            _abi.check(_abi.lib.ga3c_nccl_unique_id(uid), "ga3c_nccl_unique_id")
        if world > 1:
            import torch.distributed as dist
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0)
            C.memmove(uid, box[0], 128)
        comm = C.c_void_p(0)
        _abi.check(_abi.lib.ga3c_nccl_comm_init(world, uid, rank, device, C.byref(comm)), "ga3c_nccl_comm_init")
        self.comm = comm

    def allreduce(self, ctx, grad_from=None):
        """Sum grad_from's gradient (default ctx's) over the ranks on ctx's
        stream and recompute its non-finite flag on the sum."""
        self._abi.check(self._abi.lib.ga3c_allreduce_grads(ctx.h, grad_from.h if grad_from is not None else None,
                                                           self.comm), "ga3c_allreduce_grads")

    def close(self):
        if self.comm:
            self._abi.lib.ga3c_nccl_comm_destroy(self.comm)
            self.comm = None


def nccl_update(lp, j, U):
    """DeviceLoop data-parallel exchange over NCCL for update U (trainer
    context j): ga3c_allreduce_grads sums the gradient on the loop's main
    stream and recomputes the non-finite flag on the SUM (so every replica
    rejects or applies the same step, nnet.cpp:299-301), then the identical
    RMSProp step runs on every replica.  All on one stream: capturable."""
    lp.nccl.allreduce(lp.ctx, lp.tctx[j])
    lp.ctx.apply_slots_dev(lp.tctx[j], lp.ring[U % lp.R], lp.ring[(U + 1) % lp.R])


def peer_lists(local, gathered, rank, opener):
    """Per-rank pointer lists from every rank's {name: [pointers or handles]}:
    this rank's own pointers as they are, the peers' opened with `opener`."""
    out = {}
    for name in local:
        out[name] = [[local[name][i] if q == rank else opener(gathered[q][name][i]) for q in range(len(gathered))]
                     for i in range(len(local[name]))]
    return out


class FusedUpdate:
    """Data-parallel update through ga3c_dp_apply.  Every rank passes the
    same trainer contexts (by position) and ring slots (by id); their device
    buffers are exchanged once as CUDA IPC handles over the process group."""

    def __init__(self, model, grad_ctxs, slots, rank, world, ctas=64):
        import torch.distributed as dist

        from . import _abi
        self.dp = _abi.FusedDP(model, rank, world, ctas)
        self.slots = list(slots)
        ptrs = {"grad": [c.grad_ptr() for c in grad_ctxs],
                "theta": [_abi.slot_theta_ptr(model, sl) for sl in self.slots],
                "sig": [self.dp.signal_ptr()]}
        handles = {k: [_abi.ipc_handle(p) for p in v] for k, v in ptrs.items()}
        gathered = [None] * world
        dist.all_gather_object(gathered, handles)
        self._opened = []

        def opener(h):
            p = _abi.ipc_open(h)
            self._opened.append(p)
            return p

        self.peers = peer_lists(ptrs, gathered, rank, opener)
        self.ctxs = list(grad_ctxs)

    def apply(self, ctx, j, src_slot, dst_slot):
        """RMSProp step from src_slot into dst_slot with trainer context j's
        gradient, summed over every rank, on ctx's stream."""
        dst = self.slots.index(dst_slot)
        self.dp.apply(ctx, self.ctxs[j], src_slot, dst_slot, self.peers["grad"][j], self.peers["theta"][dst],
                      self.peers["sig"][0])

    def self_check(self, ctx, j, P, device, src, dst_fused, dst_ref):
        """One fused update against its definition, bitwise on every rank:
        all-gather every rank's gradient, sum it in rank order in fp32 (the
        order the fused kernel reduces in -- NCCL's ring/NVLS order is not
        rank order, so NCCL is not the reference here), load the sum into
        context j's gradient and run the single-GPU RMSProp kernel
        (ga3c_apply_rmsprop_slots_dev) from the same source slot.  Raises
        RuntimeError (naming the rank and the first mismatching index) if any
        rank differs; the destination slots are restored from src."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        gv = grad_view(self.ctxs[j], P, device)
        i = torch.arange(P, device=device, dtype=torch.int64)
        mine = ((((i * 7 + rank * 13) % 101) - 50).to(torch.float32) * 1e-4 * (1 + rank)).contiguous()
        from . import _abi

        def theta(slot):
            class _V:
                __cuda_array_interface__ = {"shape": (P,), "typestr": "<f4", "version": 3, "strides": None,
                                            "data": (_abi.slot_theta_ptr(self.dp.model, slot), False)}
            return torch.as_tensor(_V(), device=device)

        err = ""
        try:  # no collectives in here: a failure must not desynchronise the ranks
            gv.copy_(mine)
            torch.cuda.synchronize()
            self.apply(ctx, j, src, dst_fused)
            self.dp.check()
        except Exception as e:
            err = f"fused apply failed: {e}"
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)  # every rank, exactly once
        acc = parts[0].clone()
        for q in range(1, world):
            acc = acc + parts[q]  # fp32, rank order
        gv.copy_(acc)
        torch.cuda.synchronize()
        ctx.apply_slots_dev(self.ctxs[j], src, dst_ref)
        ctx.sync()
        a, b = theta(dst_fused), theta(dst_ref)
        if not err and not torch.equal(a, b):
            k = int(torch.nonzero(a != b)[0].item())
            err = f"theta'[{k}] fused {a[k].item()!r} != rank-order reference {b[k].item()!r}"
        ctx.copy_slot_dev(src, dst_fused)
        ctx.copy_slot_dev(src, dst_ref)
        ctx.sync()
        flag = torch.tensor([1 if err else 0], device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if flag.item():
            raise RuntimeError(f"fused DP self-check failed (rank {rank}: {err or 'ok'}; another rank failed)")
        return True

    def close(self):
        from . import _abi
        for p in self._opened:
            _abi.lib.ga3c_ipc_close(p)
        self._opened = []
        self.dp.close()
