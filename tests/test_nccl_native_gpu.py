"""The library's own NCCL data-parallel entry (ga3c_allreduce_grads,
SURVEY.md §8b) at world size 1 on the GPU box: the communicator comes up
through ga3c_nccl_unique_id / ga3c_nccl_comm_init, the all-reduce leaves the
single rank's summed gradient bit-identical, the non-finite flag is
recomputed on the result (a NaN injected after the gradient call is
rejected), and the apply that follows matches the single-GPU path."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu


def test_allreduce_grads_world_one():
    import torch

    import pyoracle as O
    from paper_1611_06256_b200 import _abi, dp

    v = C.c_int(0)
    assert _abi.lib.ga3c_nccl_version(C.byref(v)) == 0 and v.value >= 22000, v.value
    spec_o = O.make_spec((12, 12, 2), [(4, 4, 2)], [16], 3)
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(spec_o), C.sizeof(spec))
    model = _abi.Model(spec, _abi.default_hyper())
    th = O.init_model(spec_o, 5).astype(np.float32)
    model.load(th)
    ctx = _abi.Context(model, 4)
    comm = dp.NcclComm(0, 1, 0)
    fr = O.synthetic_frames(2, 4, (12, 12, 2))
    acts, rets = O.synthetic_batch(2, 4, 3)
    d_ref, _ = ctx.loss_grad(fr, acts, rets)
    comm.allreduce(ctx)
    ctx.sync()
    d_after = dp.grad_view(ctx, model.P, "cuda:0").cpu().numpy()
    assert np.array_equal(d_after, d_ref)
    ok, _ = ctx.apply_rmsprop()
    assert ok
    t1, g1, _ = model.read()
    rt, rg, _ = O.rmsprop_update_f32(O.Hyper(), th, np.zeros_like(th), d_ref)
    assert np.array_equal(t1, rt) and np.array_equal(g1, rg)
    # a non-finite value that enters after the gradient call is caught by the
    # flag recomputed on the all-reduced sum
    ctx.loss_grad(fr, acts, rets)
    gv = dp.grad_view(ctx, model.P, "cuda:0")
    gv[3] = float("nan")
    torch.cuda.synchronize()
    comm.allreduce(ctx)
    ok, _ = ctx.apply_rmsprop()
    assert not ok and model.version() == 1
    comm.close()
