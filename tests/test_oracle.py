"""Pins the CPU oracle (oracle/ga3c_oracle.c) before it is trusted as the
checker for the CUDA path.  CPU only.

  * bitwise against the reference's own nnet.cpp/returns.cpp (oracle/_ref)
    and the golden vectors generated from it (tests/golden/make_golden.py);
  * the reference's known-answer tests (test_nnet.cpp, test_returns.cpp);
  * the conv restatement: conv == dense bridge (bitwise), the reference's
    frozen-advantage finite-difference method (test_nnet.cpp:21-95) and an
    independent torch float64 autograd restatement.
"""
import math

import numpy as np
import pytest

import pyoracle as O

HYPER = O.Hyper()


# ------------------------------------------------------------ golden / ref

@pytest.mark.parametrize("name", ["ref_mlp_doc", "ref_mlp_nohidden", "ref_mlp_two", "ref_mlp_fc_tail"])
def test_oracle_matches_reference_golden_bitwise(golden, name):
    g = golden(name)
    spec = O.make_spec(int(g["input_dim"]), [], list(g["hidden"]), int(g["n_actions"]))
    th = O.init_model(spec, int(g["model_seed"]))
    if "idx" in g:
        idx = g["idx"]
        assert np.array_equal(th[idx], g["theta_sample"])
    else:
        assert np.array_equal(th, g["theta"])
    pi, v = O.forward(spec, th, g["states"])
    assert np.array_equal(pi, g["pi"]) and np.array_equal(v, g["v"])
    d, sc = O.loss_and_gradients(spec, HYPER, th, g["states"], g["actions"], g["returns"])
    assert np.array_equal(sc, g["scalars"])
    if "idx" in g:
        assert np.array_equal(d[idx], g["dtheta_sample"])
        g0 = np.abs(d) * 0.5
        to, go, ok = O.rmsprop_update(HYPER, th, g0, d)
        assert ok and np.array_equal(to[idx], g["theta_out_sample"]) and np.array_equal(go[idx], g["g_out_sample"])
    else:
        assert np.array_equal(d, g["dtheta"])
        to, go, ok = O.rmsprop_update(HYPER, th, g["g_in"], d)
        assert ok and np.array_equal(to, g["theta_out"]) and np.array_equal(go, g["g_out"])


def test_returns_match_reference_golden_bitwise(golden):
    g = golden("ref_returns")
    off = g["offsets"]
    for s in range(len(off) - 1):
        got = O.compute_returns(g["rewards"][off[s]:off[s + 1]], g["terminal"][s], g["bootstrap"][s],
                                g["gamma"][s])
        assert np.array_equal(got, g["returns"][off[s]:off[s + 1]])


def test_sampler_matches_reference_golden(golden):
    g = golden("ref_sampler")
    u = O.uniforms(int(g["seed"]), len(g["u"]))
    assert np.array_equal(u, g["u"])  # mt19937_64 + next_uniform (util.hpp:41-43)
    got = np.array([O.sample_index(g["probs"], x) for x in u])
    assert np.array_equal(got, g["actions"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("indim,hidden,A", [(4, [8], 3), (3, [], 2), (5, [6, 4], 3), (7, [5, 5, 5], 4)])
def test_oracle_matches_live_reference(indim, hidden, A):
    r = O.ref()
    hid = np.array(hidden, np.int32)
    P = r.ref_param_count(indim, hid, len(hidden), A)
    spec = O.make_spec(indim, [], hidden, A)
    assert P == O.param_count(spec)
    th = np.zeros(P)
    r.ref_init_model(indim, hid, len(hidden), A, 99, th)
    assert np.array_equal(th, O.init_model(spec, 99))
    rng = np.random.default_rng(3)
    B = 9
    st = rng.uniform(-1, 1, (B, indim))
    acts = rng.integers(0, A, B).astype(np.int32)
    rets = rng.uniform(-2, 2, B)
    for hp in (HYPER, O.Hyper(beta=0.0), O.Hyper(grad_clip_norm=0.01)):
        d = np.zeros(P)
        sc = np.zeros(3)
        r.ref_loss_and_gradients(indim, hid, len(hidden), A, hp, th, P, st, acts, rets, B, d, sc)
        d2, sc2 = O.loss_and_gradients(spec, hp, th, st, acts, rets)
        assert np.array_equal(d, d2) and np.array_equal(sc, sc2)


# ------------------------------------------------- reference known answers

def test_param_count_documented_shapes():  # test_nnet.cpp:99-106
    assert O.param_count(O.make_spec(4, [], [8], 3)) == 76
    assert O.param_count(O.make_spec(2, [], [], 2)) == 2 * 2 + 2 + 2 + 1
    assert O.param_count(O.make_spec(5, [], [7, 3], 4)) == (5 * 7 + 7) + (7 * 3 + 3) + (3 * 4 + 4) + (3 + 1)
    assert O.param_count(O.dnn_a()) == 677_943
    assert O.param_count(O.dnn_large(1)) == 4_794_503


def test_init_bounds_and_zero_biases():  # test_nnet.cpp:108-125
    th = O.init_model(O.make_spec(4, [], [8], 3), 7)
    assert np.all(np.abs(th[:32]) <= 0.5) and np.all(th[32:40] == 0)
    hb = 1 / math.sqrt(8)
    assert np.all(np.abs(th[40:64]) <= hb) and np.all(th[64:67] == 0)
    assert np.all(np.abs(th[67:75]) <= hb) and th[75] == 0


def test_rmsprop_digit_exact():  # test_nnet.cpp:237-274
    hp = O.Hyper(alpha=0.99, eta=0.1, eps_rms=1e-8)
    th = np.zeros(6); th[0] = 1.0
    d = np.zeros(6); d[0] = 2.0
    to, go, ok = O.rmsprop_update(hp, th, np.zeros(6), d)
    g = 0.99 * 0.0 + (1.0 - 0.99) * 2.0 * 2.0
    assert ok and go[0] == g and to[0] == 1.0 - 0.1 * 2.0 / math.sqrt(g + 1e-8) and to[1] == 0.0
    d2 = np.zeros(6); d2[0] = -1.0
    to2, go2, _ = O.rmsprop_update(hp, to, go, d2)
    g2 = 0.99 * g + (1.0 - 0.99) * 1.0 * 1.0
    assert go2[0] == g2 and to2[0] == to[0] + 0.1 * 1.0 / math.sqrt(g2 + 1e-8)


def test_rmsprop_rejects_nonfinite():  # test_nnet.cpp:276-291
    th = O.init_model(O.make_spec(2, [], [], 2), 3)
    g = np.zeros_like(th); g[0] = 0.5
    d = np.zeros_like(th); d[1] = np.nan
    to, go, ok = O.rmsprop_update(HYPER, th, g, d)
    assert not ok and np.array_equal(to, th) and np.array_equal(go, g)


def test_returns_known_answers():  # test_returns.cpp:37-84
    r = O.compute_returns([1.0, 0.0, 0.0, 1.0], True, 123.0, 0.99)
    assert r[3] == 1.0 and abs(r[0] - (1.0 + 0.99 * 0.9801)) < 1e-15
    assert list(O.compute_returns([0.0, 0.0], False, 10.0, 0.5)) == [2.5, 5.0]
    assert list(O.compute_returns([1.0, 1.0, 1.0], True, 0.0, 1.0)) == [3.0, 2.0, 1.0]
    for bad in (([], True, 0.0, 0.99), ([1.0], True, 0.0, 0.0), ([1.0], True, 0.0, 1.5),
                ([math.inf], True, 0.0, 0.99), ([1.0], False, math.inf, 0.99)):
        with pytest.raises(O.OracleError):
            O.compute_returns(*bad)


# ----------------------------------------------------------- conv pinning

@pytest.mark.parametrize("hw,c,hidden", [(3, 2, [8]), (5, 3, [7, 4]), (4, 4, [6])])
def test_conv_dense_bridge_bitwise(hw, c, hidden):
    """A full-size stride-1 conv is nnet::affine over the NHWC flatten: same
    layout offsets, same init draws, same summation order -> bit for bit."""
    mlp = O.make_spec(hw * hw * c, [], hidden, 3)
    conv = O.make_spec((hw, hw, c), [(hidden[0], hw, 1)], hidden[1:], 3)
    th = O.init_model(mlp, 77)
    assert np.array_equal(th, O.init_model(conv, 77))
    rng = np.random.default_rng(hw)
    st = rng.uniform(-1, 1, (6, hw * hw * c))
    acts = rng.integers(0, 3, 6).astype(np.int32)
    rets = rng.uniform(-2, 2, 6)
    assert all(np.array_equal(a, b) for a, b in zip(O.forward(mlp, th, st), O.forward(conv, th, st)))
    da, sa = O.loss_and_gradients(mlp, HYPER, th, st, acts, rets)
    db, sb = O.loss_and_gradients(conv, HYPER, th, st, acts, rets)
    assert np.array_equal(da, db) and np.array_equal(sa, sb)


def _frozen_loss(spec, hp, th, st, acts, rets, adv):
    pi, v = O.forward(spec, th, st)
    loss = 0.0
    for n in range(len(acts)):
        H = -sum(p * math.log(p + hp.eps_log) for p in pi[n])
        loss += -math.log(pi[n][acts[n]] + hp.eps_log) * adv[n] - hp.beta * H
        loss += hp.value_loss_weight * (rets[n] - v[n]) ** 2
    return loss


def test_conv_gradients_match_finite_differences():
    """test_nnet.cpp:21-95's method on a strided two-conv net."""
    spec = O.make_spec((9, 9, 2), [(3, 3, 2), (4, 2, 1)], [5], 3)
    th = O.init_model(spec, 5)
    rng = np.random.default_rng(11)
    B = 3
    st = rng.uniform(-1, 1, (B, 9 * 9 * 2))
    acts = rng.integers(0, 3, B).astype(np.int32)
    rets = rng.uniform(-2, 2, B)
    _, v = O.forward(spec, th, st)
    adv = rets - v
    d, _ = O.loss_and_gradients(spec, HYPER, th, st, acts, rets)
    worst = 0.0
    for i in range(th.size):
        h = 1e-5 * max(1.0, abs(th[i]))
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        fd = (_frozen_loss(spec, HYPER, tp, st, acts, rets, adv) -
              _frozen_loss(spec, HYPER, tm, st, acts, rets, adv)) / (2 * h)
        a = d[i]
        err = abs(a - fd) if (abs(a) < 1e-8 and abs(fd) < 1e-8) else abs(a - fd) / max(abs(a), abs(fd))
        worst = max(worst, err)
    assert worst < 1e-4


def test_conv_oracle_matches_torch_float64(golden):
    """Independent restatement with torch.nn.functional.conv2d autograd."""
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    g = golden("conv_small")
    spec = O.make_spec((12, 12, 2), [(4, 4, 2), (6, 3, 1)], [16], 3)
    th = g["theta"]
    assert np.array_equal(th, O.init_model(spec, int(g["model_seed"])))
    x = torch.tensor(O.frames_to_states(g["frames"]).reshape(-1, 12, 12, 2)).permute(0, 3, 1, 2)
    t = torch.tensor(th, requires_grad=True)
    off = 0

    def take(n):
        nonlocal off
        s = t[off:off + n]
        off += n
        return s

    h = x
    cin = 2
    for co, k, s in [(4, 4, 2), (6, 3, 1)]:
        W = take(co * k * k * cin).view(co, k, k, cin).permute(0, 3, 1, 2)
        b = take(co)
        h = F.relu(F.conv2d(h, W, b, stride=s))
        cin = co
    h = h.permute(0, 2, 3, 1).reshape(h.shape[0], -1)  # NHWC flatten
    W = take(16 * h.shape[1]).view(16, -1)
    h = F.relu(h @ W.T + take(16))
    Wp = take(3 * 16).view(3, 16)
    logits = h @ Wp.T + take(3)
    Wv = take(16).view(1, 16)
    v = (h @ Wv.T + take(1)).squeeze(1)
    pi = torch.softmax(logits, dim=1)
    assert np.allclose(pi.detach().numpy(), g["pi"], rtol=0, atol=1e-13)
    assert np.allclose(v.detach().numpy(), g["v"], rtol=0, atol=1e-13)
    acts = torch.tensor(g["actions"], dtype=torch.long)
    R = torch.tensor(g["returns"])
    adv = (R - v).detach()
    eps = HYPER.eps_log
    H = -(pi * torch.log(pi + eps)).sum(1)
    pa = pi.gather(1, acts[:, None]).squeeze(1)
    loss = (-torch.log(pa + eps) * adv - HYPER.beta * H + HYPER.value_loss_weight * (R - v) ** 2).sum()
    loss.backward()
    got = t.grad.numpy()
    ref = g["dtheta"]
    assert np.allclose(got, ref, rtol=1e-9, atol=1e-12)


def test_conv_golden_reproduces():
    import os
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "conv_small.npz")))
    spec = O.make_spec((12, 12, 2), [(4, 4, 2), (6, 3, 1)], [16], 3)
    st = O.frames_to_states(g["frames"])
    pi, v = O.forward(spec, g["theta"], st)
    d, sc = O.loss_and_gradients(spec, HYPER, g["theta"], st, g["actions"], g["returns"])
    assert np.array_equal(pi, g["pi"]) and np.array_equal(d, g["dtheta"]) and np.array_equal(sc, g["scalars"])
