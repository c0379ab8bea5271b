"""The gradient's finishing pass (final_grad_kernel): the split-K
reductions of the trunk weight gradients and the heads' weight gradient
(nnet.cpp:237-262, summed over the batch) are finished by ONE launch at the
end of the backward DAG, and the loss diagnostics by the heads kernel's
last CTA (nnet.cpp:233-235).  Checked here against the fp64 oracle at the
shapes the bench runs, on a net where EVERY weight gradient is finished by
that pass (no hidden layer), and for the reference's reject
(nnet.cpp:299-301) when the non-finite values exist only in the pieces the
pass produces.  Needs a B200 (-m gpu)."""
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


def test_conv_only_net_all_pieces_finished_in_one_pass():
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
def test_reject_when_only_finished_pieces_are_nonfinite(hidden):
    """With no hidden layer the non-finite values exist only in the pieces the
    finishing pass writes, so its flag alone must reject the step (the
    reference throws on the action, nnet.cpp:214-216, and rejects non-finite
    gradients, nnet.cpp:299-301); the device apply then leaves theta, g and
    the version unchanged."""
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
