"""Fused data-parallel update (ga3c_dp_apply, csrc/dp_fused.cuh) against the
reference semantics it replaces -- all-reduce(sum) of the per-replica summed
gradients (nnet.hpp:88-94), global non-finite reject (nnet.cpp:299-301),
clip on the reduced gradient (nnet.cpp:281-289) and RMSProp
(nnet.cpp:293-312, fp32 restatement orc_rmsprop_update_f32).

One GPU is reachable, so W ranks are W models on cuda:0 whose "peer"
pointers are the other models' raw device pointers; the rank kernels run
concurrently on their own streams and synchronise through the same signal
blocks and release/acquire protocol they use over NVLink."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu


def _setup(W, spec_o, hyper, seed=0):
    import ctypes as C

    import pyoracle as O
    from paper_1611_06256_b200 import _abi

    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(spec_o), C.sizeof(spec))
    models = [_abi.Model(spec, hyper, device=0) for _ in range(W)]
    th = O.init_model(spec_o, O.derive_seed(1, [O.SEED_MODEL_INIT])).astype(np.float32)
    rng = np.random.default_rng(seed)
    g0 = (rng.random(th.size) * 1e-3).astype(np.float32)
    for m in models:
        m.load(th, g0)
    rings = [m.ring(2) for m in models]
    ctxs = [_abi.Context(m, 4) for m in models]
    dps = [_abi.FusedDP(models[r], r, W, ctas=16) for r in range(W)]
    return models, rings, ctxs, dps, th, g0


def _grad_tensor(ctx, P):
    import torch

    from paper_1611_06256_b200 import dp
    return dp.grad_view(ctx, P, "cuda:0")


def _theta(ptr, P):
    import torch

    class _V:
        __cuda_array_interface__ = {"shape": (P,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_V(), device="cuda:0").cpu().numpy().copy()


def _step(models, ctxs, dps, src, dst, grads_np):
    import torch

    from paper_1611_06256_b200 import _abi
    W = len(models)
    P = models[0].P
    for r in range(W):
        _grad_tensor(ctxs[r], P).copy_(torch.from_numpy(grads_np[r]).cuda())
    torch.cuda.synchronize()
    gp = [c.grad_ptr() for c in ctxs]
    tp = [_abi.slot_theta_ptr(models[q], dst[q]) for q in range(W)]
    sp = [d.signal_ptr() for d in dps]
    for r in range(W):  # concurrent kernels, one per rank stream
        dps[r].apply(ctxs[r], None, src[r], dst[r], gp, tp, sp)
    for c in ctxs:
        c.sync()
    return [_theta(tp[q], P) for q in range(W)]


@pytest.mark.timeout(120)
@pytest.mark.parametrize("W", [2, 4])
def test_fused_update_bitwise_vs_allreduce_rmsprop(W):
    import pyoracle as O
    from paper_1611_06256_b200 import _abi

    spec_o = O.dnn_a()
    hyper = _abi.default_hyper()
    models, rings, ctxs, dps, th, g0 = _setup(W, spec_o, hyper)
    P = models[0].P
    rng = np.random.default_rng(1)
    g = g0
    cur = th
    for it in range(3):  # three calls: barrier epochs, sharded rms state, slot ping-pong
        grads = [(rng.standard_normal(P) * 1e-2).astype(np.float32) for _ in range(W)]
        src = [rings[r][it % 2] for r in range(W)]
        dst = [rings[r][(it + 1) % 2] for r in range(W)]
        out = _step(models, ctxs, dps, src, dst, grads)
        d = grads[0].copy()
        for q in range(1, W):
            d = (d + grads[q]).astype(np.float32)  # fixed rank order, fp32
        want_th, want_g, _ = O.rmsprop_update_f32(O.Hyper(), cur, g, d)
        for q in range(W):
            assert np.array_equal(out[q], want_th), (it, q, np.max(np.abs(out[q] - want_th)))
        cur, g = want_th, want_g


@pytest.mark.timeout(120)
def test_fused_update_nonfinite_rejected_on_every_rank():
    import pyoracle as O
    from paper_1611_06256_b200 import _abi

    W = 3
    spec_o = O.make_spec((12, 12, 2), [(4, 4, 2)], [8], 4)
    models, rings, ctxs, dps, th, g0 = _setup(W, spec_o, _abi.default_hyper())
    P = models[0].P
    grads = [np.full(P, 1e-3, np.float32) for _ in range(W)]
    grads[1][P - 3] = np.nan  # a component in the last rank's shard, produced by rank 1
    out = _step(models, ctxs, dps, [r[0] for r in rings], [r[1] for r in rings], grads)
    for q in range(W):
        assert np.array_equal(out[q], th)
    # the next call proceeds normally (epochs stay in step after a reject)
    grads = [np.full(P, 1e-3, np.float32) for _ in range(W)]
    out = _step(models, ctxs, dps, [r[1] for r in rings], [r[0] for r in rings], grads)
    d = (grads[0] + grads[1]).astype(np.float32)
    d = (d + grads[2]).astype(np.float32)
    want, _, _ = O.rmsprop_update_f32(O.Hyper(), th, g0, d)
    for q in range(W):
        assert np.array_equal(out[q], want)


@pytest.mark.timeout(120)
def test_fused_update_clips_the_reduced_gradient():
    import pyoracle as O
    from paper_1611_06256_b200 import _abi

    W = 2
    spec_o = O.make_spec((12, 12, 2), [(4, 4, 2)], [8], 4)
    hyper = _abi.default_hyper()
    hyper.grad_clip_norm = 0.05
    models, rings, ctxs, dps, th, g0 = _setup(W, spec_o, hyper)
    P = models[0].P
    rng = np.random.default_rng(3)
    grads = [(rng.standard_normal(P) * 1e-2).astype(np.float32) for _ in range(W)]
    out = _step(models, ctxs, dps, [r[0] for r in rings], [r[1] for r in rings], grads)
    d = (grads[0] + grads[1]).astype(np.float32)
    norm = np.sqrt(np.sum(d.astype(np.float64) ** 2))
    assert norm > 0.05
    dc = (d.astype(np.float64) * (0.05 / norm)).astype(np.float32)
    want, _, _ = O.rmsprop_update_f32(O.Hyper(), th, g0, dc)
    for q in range(W):
        np.testing.assert_allclose(out[q], want, rtol=1e-6, atol=1e-9)
    assert np.array_equal(out[0], out[1])  # replicas identical


@pytest.mark.timeout(120)
def test_missing_peer_times_out_instead_of_hanging():
    """Rank 1 never calls: rank 0's barrier gives up after 2 s, ga3c_dp_check
    reports it, and later calls return at once instead of waiting again."""
    import time

    import torch

    import pyoracle as O
    from paper_1611_06256_b200 import _abi

    W = 2
    spec_o = O.make_spec((12, 12, 2), [(4, 4, 2)], [8], 4)
    models, rings, ctxs, dps, th, g0 = _setup(W, spec_o, _abi.default_hyper())
    gp = [c.grad_ptr() for c in ctxs]
    tp = [_abi.slot_theta_ptr(models[q], rings[q][1]) for q in range(W)]
    sp = [d.signal_ptr() for d in dps]
    t0 = time.time()
    dps[0].apply(ctxs[0], None, rings[0][0], rings[0][1], gp, tp, sp)
    with pytest.raises(_abi.GA3CError):
        dps[0].check()
    assert 1.5 < time.time() - t0 < 30
    t1 = time.time()
    dps[0].apply(ctxs[0], None, rings[0][0], rings[0][1], gp, tp, sp)
    torch.cuda.synchronize()
    assert time.time() - t1 < 1.0
