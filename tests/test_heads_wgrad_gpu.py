"""The heads' weight gradient (nnet.cpp:237-262, summed over the batch) and
the loss diagnostics' batch sums (nnet.cpp:233-235) come from one kernel
on the backward DAG's side stream (heads_wgrad_kernel).  Checked against
the fp64 oracle at the shapes the bench runs (B = 40 at the trainer SM
budget, the predictor's 128), on a net with no hidden layer (the heads read
the conv output, D = 2592), and for the reference's reject
(nnet.cpp:299-301) of a non-finite gradient, through the device apply.
Needs a B200 (-m gpu)."""
import numpy as np
import pytest

import pyoracle as O
from test_gpu_parity import HYPER, grad_close, make, theta32

pytestmark = pytest.mark.gpu


def case(spec, B, seed, budget=0, bad_action=False):
    m, ctx = make(spec, max_batch=B)
    th = theta32(spec, O.derive_seed(seed, [O.SEED_MODEL_INIT]))
    m.load(th)
    ctx.set_sm_budget(budget)
    fr = O.synthetic_frames(seed + 7, B)
    acts, rets = O.synthetic_batch(seed + 3, B, spec.n_actions)
    if bad_action:
        acts = acts.copy()
        acts[B // 2] = spec.n_actions  # out of range: NaN advantage, every gradient piece non-finite
    return m, ctx, th, fr, acts, rets


@pytest.mark.parametrize("B,budget", [(40, 0), (40, 111), (5, 0), (128, 0)])
def test_dnn_a_gradient_and_scalars(B, budget):
    spec = O.dnn_a()
    m, ctx, th, fr, acts, rets = case(spec, B, 11, budget)
    d1, s1 = ctx.loss_grad(fr, acts, rets)
    d2, s2 = ctx.loss_grad(fr, acts, rets)
    assert np.array_equal(d1, d2) and np.array_equal(s1, s2)  # fixed-order, run to run
    rd, rsc = O.loss_and_gradients(spec, HYPER, th.astype(np.float64), O.frames_to_states(fr), acts, rets)
    grad_close(d1, rd)
    # the loss sum cancels (terms of both signs): fp32-level error per sample
    assert np.allclose(s1, rsc, rtol=1e-5, atol=1e-6 * B), (s1, rsc)


def test_conv_only_net_wide_heads():
    spec = O.make_spec((84, 84, 4), [(16, 8, 4), (32, 4, 2)], [], 6)
    m, ctx, th, fr, acts, rets = case(spec, 40, 2)
    d, sc = ctx.loss_grad(fr, acts, rets)
    rd, rsc = O.loss_and_gradients(spec, HYPER, th.astype(np.float64), O.frames_to_states(fr), acts, rets)
    grad_close(d, rd)
    assert np.allclose(sc, rsc, rtol=1e-5, atol=1e-6)


def test_large1_batch8():
    spec = O.dnn_large(1)
    m, ctx, th, fr, acts, rets = case(spec, 8, 4)
    d, sc = ctx.loss_grad(fr, acts, rets)
    rd, rsc = O.loss_and_gradients(spec, HYPER, th.astype(np.float64), O.frames_to_states(fr), acts, rets)
    grad_close(d, rd)


@pytest.mark.parametrize("hidden", [[256], []])
def test_reject_nonfinite_through_device_apply(hidden):
    """An out-of-range action (the reference throws, nnet.cpp:214-216) makes
    every gradient piece non-finite; the device apply then rejects the step
    (nnet.cpp:299-301) and leaves theta, g and the version unchanged."""
    import torch
    spec = O.make_spec((84, 84, 4), [(16, 8, 4), (32, 4, 2)], hidden, 6)
    m, ctx, th, fr, acts, rets = case(spec, 40, 9, bad_action=True)
    src, dst = m.ring(2)
    d_fr = torch.as_tensor(fr).cuda()
    d_a = torch.as_tensor(acts.astype(np.int32)).cuda()
    d_r = torch.as_tensor(rets.astype(np.float64)).cuda()
    ctx.loss_grad_dev(d_fr.data_ptr(), True, d_a.data_ptr(), d_r.data_ptr(), 40, src)
    v0 = ctx.dev_version()
    ctx.apply_slots_dev(ctx, src, dst)
    ctx.sync()
    d, _ = ctx.read_grad()
    assert not np.isfinite(d).all()
    t0, g0 = m.read_slot(src)
    t1, g1 = m.read_slot(dst)
    assert np.array_equal(t1, t0) and np.array_equal(g1, g0) and ctx.dev_version() == v0
    # the control words are back at rest: a clean step applies
    d_a.zero_()
    ctx.loss_grad_dev(d_fr.data_ptr(), True, d_a.data_ptr(), d_r.data_ptr(), 40, src)
    ctx.apply_slots_dev(ctx, src, dst)
    ctx.sync()
    d, _ = ctx.read_grad()
    rt, rg, _ = O.rmsprop_update_f32(HYPER, t0, g0, d)
    t2, g2 = m.read_slot(dst)
    assert np.array_equal(t2, rt) and np.array_equal(g2, rg) and ctx.dev_version() == v0 + 1
