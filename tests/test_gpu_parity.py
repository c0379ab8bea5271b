"""Parity of the CUDA path (through the C ABI) with the CPU oracle on the same
seeded inputs.  Needs a B200: run with -m gpu.

Tolerances (fp32 device arithmetic vs the fp64 reference):
  pi            max |d|            <= 2e-6
  V             max |d| / max|V|   <= 1e-5
  dtheta        ||d||_2 / ||ref||_2 <= 1e-5, and per component
                |d| <= 1e-4 * max|ref| + 1e-3 * |ref|
  loss scalars  relative            <= 1e-5
  RMSProp       BITWISE vs the fp32 restatement orc_rmsprop_update_f32, and
                |d| <= 1e-6 + 1e-5 |theta'| vs fp64 rmsprop_update
  returns       BITWISE (fp64, reference operation order)
  sampled actions BITWISE vs util.hpp:46-54 on the oracle's policy with the
                same u stream (draws within 1e-9 of a CDF boundary are
                counted and must be zero)
"""
import ctypes as C

import numpy as np
import pytest

import pyoracle as O

pytestmark = pytest.mark.gpu

HYPER = O.Hyper()


def abi():
    from paper_1611_06256_b200 import _abi
    return _abi


def make(spec, hyper=HYPER, max_batch=64):
    _abi = abi()
    s = _abi.NetSpec()
    C.memmove(C.byref(s), C.byref(spec), C.sizeof(s))
    h = _abi.HyperC()
    C.memmove(C.byref(h), C.byref(hyper), C.sizeof(h))
    m = _abi.Model(s, h)
    return m, _abi.Context(m, max_batch)


def theta32(spec, seed):
    return O.init_model(spec, seed).astype(np.float32)


def check_forward(spec, th32, states_dev, states_orc):
    m, ctx = make(spec, max_batch=max(1, len(states_orc)))
    m.load(th32)
    pi, v, ver = ctx.forward(states_dev)
    rpi, rv = O.forward(spec, th32.astype(np.float64), states_orc)
    assert ver == 0
    assert np.max(np.abs(pi - rpi)) <= 2e-6, np.max(np.abs(pi - rpi))
    assert np.max(np.abs(v - rv)) <= 1e-5 * max(1.0, np.max(np.abs(rv))), np.max(np.abs(v - rv))
    assert np.allclose(pi.sum(1), 1.0, atol=1e-6)
    return m, ctx


def grad_close(got, ref):
    got = got.astype(np.float64)
    rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert rel <= 1e-5, rel
    tol = 1e-4 * np.max(np.abs(ref)) + 1e-3 * np.abs(ref)
    bad = np.abs(got - ref) > tol
    assert not bad.any(), (np.flatnonzero(bad)[:10], got[bad][:5], ref[bad][:5])


def check_grad(spec, th32, states_dev, states_orc, acts, rets, hyper=HYPER):
    m, ctx = make(spec, hyper, max_batch=len(acts))
    m.load(th32)
    d, sc = ctx.loss_grad(states_dev, acts, rets)
    rd, rsc = O.loss_and_gradients(spec, hyper, th32.astype(np.float64), states_orc, acts, rets)
    grad_close(d, rd)
    assert np.allclose(sc, rsc, rtol=1e-5, atol=1e-6), (sc, rsc)
    return d


# ------------------------------------------------------------------ DNN A

@pytest.mark.parametrize("B", [1, 5, 32])
def test_dnn_a_forward(B):
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    fr = O.synthetic_frames(10 + B, B)
    check_forward(spec, th, fr, O.frames_to_states(fr))


@pytest.mark.parametrize("B", [1, 5, 20])
def test_dnn_a_loss_and_gradients(B):
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    fr = O.synthetic_frames(20 + B, B)
    acts, rets = O.synthetic_batch(20 + B, B, 6)
    check_grad(spec, th, fr, O.frames_to_states(fr), acts, rets)


# B >= 95 frames is >= 2 tiles per SM: conv1 runs the persistent int8 kernel
# (tc_u8conv.cuh) -- tiles straddling two frames, multi-tile CTAs, the TMA
# footprint ring wrapping around.
@pytest.mark.parametrize("B", [128, 256])
def test_dnn_a_forward_persistent_conv1(B):
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    fr = O.synthetic_frames(40 + B, B)
    check_forward(spec, th, fr, O.frames_to_states(fr))


def test_dnn_a_loss_and_gradients_persistent_conv1():
    B = 128
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    fr = O.synthetic_frames(50, B)
    acts, rets = O.synthetic_batch(50, B, 6)
    check_grad(spec, th, fr, O.frames_to_states(fr), acts, rets)


def test_large_dnn_stride1_forward_persistent_conv1():
    spec = O.dnn_large(1)  # 77x77 conv1 outputs: 371 tiles at B = 8, odd rows straddle tiles
    th = theta32(spec, 3)
    fr = O.synthetic_frames(6, 8)
    check_forward(spec, th, fr, O.frames_to_states(fr))


def test_large_dnn_stride1_batch16_forward_and_gradients():
    """B = 16: conv2's 171 tiles exceed the SMs (multi-wave, shallow rings),
    every weight gradient splits over many CTAs."""
    spec = O.dnn_large(1)
    th = theta32(spec, 3)
    fr = O.synthetic_frames(7, 16)
    st = O.frames_to_states(fr)
    check_forward(spec, th, fr, st)
    acts, rets = O.synthetic_batch(7, 16, 6)
    check_grad(spec, th, fr, st, acts, rets)


def test_dnn_a_golden(golden):
    g = golden("dnn_a")
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    m, ctx = make(spec, max_batch=8)
    m.load(th)
    pi, v, _ = ctx.forward(g["frames"])
    assert np.max(np.abs(pi - g["pi"])) <= 2e-6
    d, sc = ctx.loss_grad(g["frames"], g["actions"], g["returns"])
    ref = g["dtheta_sample"]
    got = d[g["idx"]].astype(np.float64)
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
    assert abs(np.linalg.norm(d.astype(np.float64)) - g["dtheta_norm"]) <= 1e-5 * g["dtheta_norm"]
    assert np.allclose(sc, g["scalars"], rtol=1e-5)


def test_large_dnn_stride4():
    spec = O.dnn_large(4)
    th = theta32(spec, 3)
    fr = O.synthetic_frames(4, 3)
    st = O.frames_to_states(fr)
    check_forward(spec, th, fr, st)
    acts, rets = O.synthetic_batch(4, 3, 6)
    check_grad(spec, th, fr, st, acts, rets)


@pytest.mark.slow
def test_large_dnn_stride1():
    spec = O.dnn_large(1)
    th = theta32(spec, 3)
    fr = O.synthetic_frames(5, 2)
    st = O.frames_to_states(fr)
    check_forward(spec, th, fr, st)
    acts, rets = O.synthetic_batch(5, 2, 6)
    check_grad(spec, th, fr, st, acts, rets)


@pytest.mark.parametrize("sms", [0, 111])
def test_large1_bench_batches(sms):
    """large s1 at the batch sizes its bench line runs: predictor forward at
    B = 128 (the persistent int8 conv1 path) and loss/backward at B = 40,
    against the oracle (threaded over the batch); whole-GPU plans (the
    large-net default) and the shared 111-SM trainer plan."""
    spec = O.dnn_large(1)
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    m, ctx = make(spec, max_batch=128)
    m.load(th)
    ctx.set_sm_budget(sms)
    fr = O.synthetic_frames(11, 128)
    st = O.frames_to_states(fr)
    pi, v, _ = ctx.forward(fr)
    rpi, rv = O.forward_mt(spec, th.astype(np.float64), st)
    assert np.max(np.abs(pi - rpi)) <= 2e-6, np.max(np.abs(pi - rpi))
    assert np.max(np.abs(v - rv)) <= 1e-5 * max(1.0, np.max(np.abs(rv)))
    acts, rets = O.synthetic_batch(11, 40, 6)
    d, sc = ctx.loss_grad(fr[:40], acts, rets)
    rd, rsc = O.loss_and_gradients_mt(spec, HYPER, th.astype(np.float64), st[:40], acts, rets)
    grad_close(d, rd)
    assert np.allclose(sc, rsc, rtol=1e-5, atol=1e-6), (sc, rsc)


BAND_CASES = [
    # (spec, B, SM budget): the u8 first-layer weight gradient staged per
    # image (tc_wgrad_band.cuh) -- k * Cin == 32 window rows
    (O.dnn_a(), 1, 2),                      # one CTA, one split: dtheta stored directly
    (O.dnn_a(), 3, 0),                      # whole GPU: 13 CTAs per image, one chunk each
    (O.dnn_a(), 40, 111),                   # the bench's trainer plan: one CTA per image
    (O.dnn_a(), 40, 16),                    # a small budget: one CTA per image as well
    (O.make_spec((20, 20, 8), [(8, 4, 2)], [16], 4), 5, 0),   # k = 4: one 128-kk tile (MT = 1)
    (O.make_spec((32, 32, 4), [(12, 8, 3)], [32], 5), 7, 0),  # stride 3, P = 81, 12 filters
]


@pytest.mark.parametrize("case", range(len(BAND_CASES)))
def test_band_first_layer_weight_gradient(case):
    """The staged-band conv1 weight gradient against the fp64 oracle
    (nnet.cpp:58-73, 262-278) over its plans: direct store, many CTAs per
    image with one chunk each, one CTA per image, a single 128-kk tile, an
    odd stride and pixel count; deterministic run to run."""
    spec, B, budget = BAND_CASES[case]
    H, W, Cc = spec.in_h, spec.in_w, spec.in_c
    th = theta32(spec, 40 + case)
    fr = O.synthetic_frames(50 + case, B, (H, W, Cc))
    st = O.frames_to_states(fr)
    acts, rets = O.synthetic_batch(60 + case, B, spec.n_actions)
    m, ctx = make(spec, max_batch=B)
    m.load(th)
    ctx.set_sm_budget(budget)
    d1, s1 = ctx.loss_grad(fr.reshape(B, -1), acts, rets)
    d2, s2 = ctx.loss_grad(fr.reshape(B, -1), acts, rets)
    assert np.array_equal(d1, d2) and np.array_equal(s1, s2)
    rd, rsc = O.loss_and_gradients(spec, HYPER, th.astype(np.float64), st, acts, rets)
    grad_close(d1, rd)
    assert np.allclose(s1, rsc, rtol=1e-5, atol=1e-6), (s1, rsc)


def test_conv_small_golden(golden):
    g = golden("conv_small")
    spec = O.make_spec((12, 12, 2), [(4, 4, 2), (6, 3, 1)], [16], 3)
    # the golden was produced on fp64 weights: compare against the oracle on
    # the fp32-rounded weights the device uses, and loosely against the file
    th = g["theta"].astype(np.float32)
    st = O.frames_to_states(g["frames"])
    check_forward(spec, th, g["frames"], st)
    d = check_grad(spec, th, g["frames"], st, g["actions"], g["returns"])
    assert np.linalg.norm(d - g["dtheta"]) <= 1e-5 * np.linalg.norm(g["dtheta"])


# ---------------------------------------------- reference MLP golden cases

@pytest.mark.parametrize("name", ["ref_mlp_doc", "ref_mlp_nohidden", "ref_mlp_two", "ref_mlp_fc_tail"])
def test_reference_mlp_golden(golden, name):
    g = golden(name)
    spec = O.make_spec(int(g["input_dim"]), [], list(g["hidden"]), int(g["n_actions"]))
    th = O.init_model(spec, int(g["model_seed"])).astype(np.float32)
    st = g["states"].astype(np.float32)
    st64 = st.astype(np.float64)
    check_forward(spec, th, st, st64)
    check_grad(spec, th, st, st64, g["actions"], g["returns"])


@pytest.mark.parametrize("hyper", [O.Hyper(beta=0.0), O.Hyper(grad_clip_norm=0.01), O.Hyper(value_loss_weight=2.0)])
def test_hyperparameter_variants(hyper):
    spec = O.make_spec((12, 12, 2), [(4, 4, 2)], [8], 4)
    th = theta32(spec, 8)
    fr = O.synthetic_frames(8, 6, (12, 12, 2))
    acts, rets = O.synthetic_batch(8, 6, 4)
    check_grad(spec, th, fr, O.frames_to_states(fr), acts, rets, hyper)


def test_gradients_summed_not_averaged():  # test_nnet.cpp:175-189
    spec = O.make_spec(4, [], [8], 3)
    m, ctx = make(spec)
    m.load(theta32(spec, 5))
    st = np.array([[0.1, -0.2, 0.3, 0.4]], np.float32)
    d1, _ = ctx.loss_grad(st, [1], [0.7])
    d2, _ = ctx.loss_grad(np.repeat(st, 2, 0), [1, 1], [0.7, 0.7])
    assert np.allclose(d2, 2 * d1, rtol=1e-6, atol=1e-12)


def test_collapsed_policy_gradient_finite():  # test_nnet.cpp:191-227
    spec = O.make_spec(2, [], [], 2)
    th = np.zeros(O.param_count(spec), np.float32)
    th[0] = 40.0
    th[3] = 40.0
    m, ctx = make(spec)
    m.load(th)
    pi, _, _ = ctx.forward(np.array([[1.0, 0.0]], np.float32))
    assert pi[0, 1] < 1e-15
    d, _ = ctx.loss_grad(np.array([[1.0, 0.0]], np.float32), [1], [2.0])
    assert np.all(np.isfinite(d))


# ------------------------------------------------------------------ RMSProp

def test_rmsprop_bitwise_vs_fp32_restatement():
    spec = O.dnn_a()
    P = O.param_count(spec)
    rng = np.random.default_rng(0)
    th = theta32(spec, 1)
    g = (rng.random(P, np.float32) * 1e-3).astype(np.float32)
    d = (rng.standard_normal(P) * 1e-2).astype(np.float32)
    m, ctx = make(spec)
    m.load(th, g, 41)
    ok, on = ctx.apply_rmsprop(d)
    assert ok and on == 41
    th2, g2, ver = m.read()
    assert ver == 42
    rt, rg, rok = O.rmsprop_update_f32(HYPER, th, g, d)
    assert rok and np.array_equal(th2, rt) and np.array_equal(g2, rg)
    t64, g64, _ = O.rmsprop_update(HYPER, th.astype(np.float64), g.astype(np.float64), d.astype(np.float64))
    assert np.all(np.abs(th2 - t64) <= 1e-6 + 1e-5 * np.abs(t64))


def test_rmsprop_digit_test_on_device():  # test_nnet.cpp:237-274 (fp32 restated)
    hyper = O.Hyper(alpha=0.99, eta=0.1, eps_rms=1e-8)
    spec = O.make_spec(1, [], [], 2)
    m, ctx = make(spec, hyper)
    th = np.zeros(6, np.float32)
    th[0] = 1.0
    m.load(th)
    d = np.zeros(6, np.float32)
    d[0] = 2.0
    assert ctx.apply_rmsprop(d) == (True, 0)
    t1, g1, v1 = m.read()
    rt, rg, _ = O.rmsprop_update_f32(hyper, th, np.zeros(6, np.float32), d)
    assert np.array_equal(t1, rt) and np.array_equal(g1, rg) and v1 == 1 and t1[1] == 0.0
    assert abs(g1[0] - 0.04) <= 1e-8 and abs(t1[0] - (1 - 0.1 * 2 / np.sqrt(0.04 + 1e-8))) <= 1e-6
    d2 = np.zeros(6, np.float32)
    d2[0] = -1.0
    ctx.apply_rmsprop(d2)
    t2, g2, v2 = m.read()
    rt2, rg2, _ = O.rmsprop_update_f32(hyper, t1, g1, d2)
    assert np.array_equal(t2, rt2) and np.array_equal(g2, rg2) and v2 == 2


def test_rmsprop_rejects_nonfinite_and_keeps_version():  # test_nnet.cpp:276-291
    spec = O.make_spec(2, [], [], 2)
    m, ctx = make(spec)
    th = theta32(spec, 3)
    g = np.zeros_like(th)
    g[0] = 0.5
    m.load(th, g, 7)
    d = np.zeros_like(th)
    d[1] = np.nan
    assert ctx.apply_rmsprop(d) == (False, None)
    t2, g2, v = m.read()
    assert np.array_equal(t2, th) and np.array_equal(g2, g) and v == 7


def test_snapshot_is_immutable_across_apply():  # pipeline.hpp:87-91, test_pipeline.cpp:100-121
    spec = O.make_spec(4, [], [8], 3)
    m, ctx = make(spec)
    th = theta32(spec, 9)
    m.load(th)
    slot, ver = m.acquire()
    st = np.array([[0.5, 0.0, -0.5, 1.0]], np.float32)
    pi0, _, _ = ctx.forward(st, slot=slot)
    ctx.loss_grad(st, [2], [1.5], slot=slot, want_grad=False)
    ok, on = ctx.apply_rmsprop()  # gradient of snapshot v applied on the latest
    assert ok and on == 0 and m.version() == 1
    pi1, _, ver_used = ctx.forward(st, slot=slot)  # pinned snapshot still v0
    assert np.array_equal(pi0, pi1)
    m.release(slot)
    pi2, _, v2 = ctx.forward(st)
    assert v2 == 1 and not np.array_equal(pi0, pi2)


# ---------------------------------------------------------- returns / sampling

def test_returns_bitwise(golden):
    g = golden("ref_returns")
    spec = O.make_spec(1, [], [], 2)
    _, ctx = make(spec)
    off = g["offsets"]
    # the kernel takes one gamma per call: group segments by gamma
    for s in range(len(off) - 1):
        out = ctx.compute_returns(g["rewards"][off[s]:off[s + 1]], [0, off[s + 1] - off[s]],
                                  [g["terminal"][s]], [g["bootstrap"][s]], g["gamma"][s])
        assert np.array_equal(out, g["returns"][off[s]:off[s + 1]])
    # batched: all segments with gamma 0.99 at once
    r = np.concatenate([g["rewards"][off[s]:off[s + 1]] for s in range(len(off) - 1)])
    out = ctx.compute_returns(r, off, g["terminal"], g["bootstrap"], 0.99)
    for s in range(len(off) - 1):
        want = O.compute_returns(g["rewards"][off[s]:off[s + 1]], g["terminal"][s], g["bootstrap"][s], 0.99)
        assert np.array_equal(out[off[s]:off[s + 1]], want)


def test_returns_validation():
    spec = O.make_spec(1, [], [], 2)
    _, ctx = make(spec)
    with pytest.raises(ValueError):
        ctx.compute_returns([1.0], [0, 1], [1], [0.0], 0.0)
    with pytest.raises(ValueError):
        ctx.compute_returns([np.inf], [0, 1], [1], [0.0], 0.9)
    with pytest.raises(ValueError):
        ctx.compute_returns([1.0], [0, 1], [0], [np.nan], 0.9)
    assert list(ctx.compute_returns([1.0], [0, 1], [1], [np.nan], 0.5)) == [1.0]


def test_sampled_actions_bitwise():
    torch = pytest.importorskip("torch")
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    B = 256
    fr = O.synthetic_frames(77, B)
    rpi, _ = O.forward(spec, th.astype(np.float64), O.frames_to_states(fr))
    u = O.uniforms(O.derive_seed(1, [O.SEED_AGENT_RNG, 0]), B)
    want = np.array([O.sample_index(rpi[b], u[b]) for b in range(B)])
    cdf = np.cumsum(rpi, 1)
    margin = np.min(np.abs(cdf - u[:, None]))
    assert margin > 1e-9  # no draw sits on a CDF boundary
    m, ctx = make(spec, max_batch=B)
    m.load(th)
    dfr = torch.from_numpy(fr).cuda()
    du = torch.from_numpy(u).cuda()
    dact = torch.zeros(B, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx.forward_dev(dfr.data_ptr(), B, True)
    ctx.sample_dev(du.data_ptr(), B, dact.data_ptr())
    ctx.sync()
    assert np.array_equal(dact.cpu().numpy(), want)


# ---------------------------------------------------------------- validation

def test_input_validation_matches_reference():
    spec = O.make_spec(2, [], [], 2)
    m, ctx = make(spec)
    m.load(theta32(spec, 1))
    with pytest.raises(ValueError):
        ctx.forward(np.array([[1.0, np.nan]], np.float32))
    with pytest.raises(ValueError):
        ctx.loss_grad(np.zeros((1, 2), np.float32), [5], [0.0])
    with pytest.raises(ValueError):
        ctx.loss_grad(np.zeros((1, 2), np.float32), [0], [np.inf])
    with pytest.raises(ValueError):
        ctx.loss_grad(np.zeros((0, 2), np.float32), [], [])
    pi, v, _ = ctx.forward(np.zeros((0, 2), np.float32))
    assert pi.shape == (0, 2)


def test_deterministic_gradients():
    spec = O.dnn_a()
    th = theta32(spec, 2)
    fr = O.synthetic_frames(3, 16)
    acts, rets = O.synthetic_batch(3, 16, 6)
    m, ctx = make(spec, max_batch=16)
    m.load(th)
    d1, s1 = ctx.loss_grad(fr, acts, rets)
    d2, s2 = ctx.loss_grad(fr, acts, rets)
    assert np.array_equal(d1, d2) and np.array_equal(s1, s2)


@pytest.mark.parametrize("sms", [16, 49])
def test_sm_budget_changes_plans_not_results(sms):
    """ga3c_ctx_set_sm_budget re-plans every split-K (fewer, longer CTAs);
    the gradient stays within the parity tolerance of the oracle and is
    deterministic for a given budget."""
    B = 40
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    fr = O.synthetic_frames(60, B)
    acts, rets = O.synthetic_batch(60, B, 6)
    m, ctx = make(spec, max_batch=B)
    m.load(th)
    ctx.set_sm_budget(sms)
    d1, _ = ctx.loss_grad(fr, acts, rets)
    d2, _ = ctx.loss_grad(fr, acts, rets)
    assert np.array_equal(d1, d2)
    rd, _ = O.loss_and_gradients(spec, HYPER, th.astype(np.float64), O.frames_to_states(fr), acts, rets)
    grad_close(d1, rd)


def test_stream_priority_changes_scheduling_not_results():
    """ga3c_ctx_set_priority re-creates the context stream one or more
    levels lower (the trainer pool's and engine's trainers run at level 1);
    forward and gradient are bitwise what the default-priority context
    computes, and a level past the device's range clamps to the lowest."""
    B = 40
    spec = O.dnn_a()
    th = theta32(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    fr = O.synthetic_frames(61, B)
    acts, rets = O.synthetic_batch(61, B, 6)
    m, ctx = make(spec, max_batch=B)
    m.load(th)
    d0, s0 = ctx.loss_grad(fr, acts, rets)
    p0, v0, _ = ctx.forward(fr)
    old = ctx.stream
    for level in (1, 1000, 0):
        ctx.set_priority(level)
        d1, s1 = ctx.loss_grad(fr, acts, rets)
        p1, v1, _ = ctx.forward(fr)
        assert np.array_equal(d0, d1) and np.array_equal(s0, s1)
        assert np.array_equal(p0, p1) and np.array_equal(v0, v1)
    assert ctx.stream != 0 and old != 0
    from paper_1611_06256_b200 import _abi
    with pytest.raises(_abi.GA3CError):
        ctx.set_priority(-1)


def test_copy_slot_publishes_parameters():
    spec = O.make_spec((12, 12, 2), [(4, 4, 2)], [8], 4)
    m, ctx = make(spec, max_batch=4)
    th = theta32(spec, 5)
    m.load(th)
    a, b = m.ring(2)
    from paper_1611_06256_b200 import _abi
    import torch
    ctx.copy_slot_dev(a, b)
    ctx.sync()

    class _V:
        __cuda_array_interface__ = {"shape": (m.P,), "typestr": "<f4", "version": 3, "strides": None,
                                    "data": (_abi.slot_theta_ptr(m, b), False)}
    assert np.array_equal(torch.as_tensor(_V(), device="cuda").cpu().numpy(), th)


def test_apply_rmsprop_dev_in_place_and_reject():
    """ga3c_apply_rmsprop_dev (the graph-capturable in-place apply) matches the
    fp32 restatement bitwise on the context gradient, and a non-finite
    gradient leaves theta, g and the version untouched (nnet.cpp:299-301;
    the kernel issues the reject-flag load beside the data loads)."""
    spec = O.make_spec(4, [], [8], 3)
    m, ctx = make(spec)
    th = theta32(spec, 11)
    m.load(th)
    st = np.array([[0.5, 0.0, -0.5, 1.0], [1.0, -1.0, 0.25, 0.0]], np.float32)
    d, _ = ctx.loss_grad(st, [2, 0], [1.5, -0.5])
    v0 = ctx.dev_version()
    ctx.apply_rmsprop_dev()
    t1, g1, _ = m.read()
    rt, rg, _ = O.rmsprop_update_f32(HYPER, th, np.zeros_like(th), d)
    # the device loop counts its updates on the device (no host publish)
    assert np.array_equal(t1, rt) and np.array_equal(g1, rg) and ctx.dev_version() == v0 + 1
    # overflow to inf in the forward pass -> non-finite gradient -> rejected
    big = np.full((1, 4), 3e38, np.float32)
    ctx.loss_grad(big, [1], [1.0], want_grad=False)
    ctx.apply_rmsprop_dev()
    t2, g2, _ = m.read()
    assert np.array_equal(t2, t1) and np.array_equal(g2, g1) and ctx.dev_version() == v0 + 1


@pytest.mark.parametrize("B", [4, 40])
def test_tma_conv_forward_cluster_and_channel_offsets(B):
    """The TMA-staged conv forward (im2col tensor map over the NHWC input +
    tiled weight map, tc_kk_ws_kernel<..., TMA>): Cin = 32 and 64 layers
    (a 64-channel input takes two 32-channel boxes per filter tap), a 3x3
    stride-1 window, and grids small enough that K is split over a cluster
    (DSMEM reduction) -- forward and gradients against the oracle."""
    spec = O.make_spec((84, 84, 4), [(32, 8, 4), (64, 4, 2), (64, 3, 1)], [64], 6)
    th = theta32(spec, 21)
    fr = O.synthetic_frames(5, B)
    st = O.frames_to_states(fr)
    check_forward(spec, th, fr, st)
    acts, rets = O.synthetic_batch(5, B, 6)
    check_grad(spec, th, fr, st, acts, rets)
