"""Parity of the EXACT benchmarked configuration with the oracle.

bench.py times paper_1611_06256_b200.loop.DeviceLoop: DNN A, N_A = 128
agents, t_max = 5, min_train_batch = 40 (16 updates per step), N_T = 3
trainer contexts in flight over a ring of 4 parameter slots, trainer SM
budget 111 and predictor SM budget 64 (the bench's automatic budgets for
DNN A), the predictor of step i beside the trainers of step i (which
consume step i-1's experiences), and CUDA graphs chaining steps.  This test
builds that loop with the same code, replays ONE captured graph of two
chained steps (32 updates), and has the fp64 oracle execute the same
version schedule:

  update U's gradient is taken on version max(0, U - N_T + 1) and applied
  on top of version U (loop.grad_version), the batch of update u of step i
  being samples [40u, 40u + 40) of step i-1's agent-major experiences.

Checked:
  * the predictor's sampled actions of step 0 equal qac::sample_index
    (util.hpp:46-54) on the oracle's policy with the same uniforms (draws
    within 1e-6 of a CDF boundary are counted and reported);
  * the step-0 n-step returns within 1e-5 of the oracle's (returns.cpp:8-26,
    bootstrapped with the oracle's own V);
  * theta and the RMSProp accumulator g after 32 updates against the
    oracle's fp64 trajectory: max |dtheta| <= 1e-5 and <= 1e-3 of the total
    parameter movement ||theta_32 - theta_0||_inf; g relative to max g <= 2e-4
    (measured on B200: 2.5e-7, 1.2e-5 of the movement, g 1.4e-5).
    (fp32 device arithmetic with 3xTF32 GEMMs; RMSProp's normalised steps
    carry the gradient's ~1e-6 relative error into theta at ~eta per update.)
"""
import ctypes as C

import numpy as np
import pytest

import pyoracle as O

pytestmark = pytest.mark.gpu

NA, T, TB, NT = 128, 5, 40, 3
TRAINER_SMS, PRED_SMS = 111, 64


def _inputs(sets, seed=7):
    rng = np.random.default_rng(seed)
    frames = rng.integers(0, 256, (sets, NA, T, 84, 84, 4), dtype=np.uint8)
    uni = rng.random((sets, T, NA))
    rewards = rng.random((sets, NA, T)) * 2 - 1
    terminal = (rng.random((sets, NA)) < T / 64.0).astype(np.uint8)
    return frames, uni, rewards, terminal


def test_headline_schedule_matches_oracle():
    import torch

    from paper_1611_06256_b200 import _abi
    from paper_1611_06256_b200.loop import DeviceLoop, grad_version

    spec_o = O.dnn_a()
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(spec_o), C.sizeof(spec))
    hyper = _abi.default_hyper()
    model = _abi.Model(spec, hyper)
    ctx = _abi.Context(model, NA)
    th0 = O.init_model(spec_o, O.derive_seed(1, [O.SEED_MODEL_INIT])).astype(np.float32)
    model.load(th0)

    sets = 2
    frames, uni, rewards, terminal = _inputs(sets)
    dev = lambda a: torch.from_numpy(a).cuda()
    loop = DeviceLoop(model, ctx, NA, T, TB, NT, dev(frames), dev(uni), dev(rewards), dev(terminal),
                      trainer_sms=TRAINER_SMS, pred_sms=PRED_SMS, overlap=True, hyper=hyper)
    graphs, _ = loop.capture(G=2)  # graph 0 = steps 0, 1 (updates 0..31, continuous)
    loop.launch(graphs[0])
    loop.sync()
    torch.cuda.synchronize()
    th_dev, g_dev = model.read_slot(loop.latest_slot())
    acts0 = loop.actions2[0].cpu().numpy()  # step 0's experiences, consumed by step 1
    rets0 = loop.rets2[0].cpu().numpy()

    # ---- oracle: step 0's predictor on version 0 (frames of set 0)
    th = th0.astype(np.float64)
    st0 = O.frames_to_states(frames[0].reshape(NA * T, 84, 84, 4)).reshape(NA, T, -1)
    near = 0
    v_last = None
    for t in range(T):
        pi, v = O.forward_mt(spec_o, th, st0[:, t])
        for b in range(NA):
            cdf = np.cumsum(pi[b])
            near += int(np.any(np.abs(cdf - uni[0, t, b]) < 1e-6))
            want = O.sample_index(pi[b], uni[0, t, b])
            assert acts0[b, t] == want, (t, b, acts0[b, t], want, pi[b], uni[0, t, b])
        v_last = v
    print(f"sampled actions: {NA * T} equal, {near} draws within 1e-6 of a CDF boundary")
    rets_o = np.stack([O.compute_returns(rewards[0, a], bool(terminal[0, a]), 0.0 if terminal[0, a] else v_last[a],
                                         hyper.gamma) for a in range(NA)])
    assert np.max(np.abs(rets0 - rets_o)) <= 1e-5 * max(1.0, np.max(np.abs(rets_o))), np.max(np.abs(rets0 - rets_o))

    # ---- oracle: the 32 updates of the version schedule
    hp = O.Hyper()
    updates = NA * T // TB
    versions = [th]
    g = np.zeros_like(th)
    # step 0 trains on the (zero-initialised) buffer of "step -1": frames of
    # set (0 - 1) % sets, action 0, return 0; step 1 on step 0's experiences
    batches = [(O.frames_to_states(frames[1].reshape(NA * T, 84, 84, 4)), np.zeros(NA * T, np.int32),
                np.zeros(NA * T)),
               (st0.reshape(NA * T, -1), acts0.reshape(-1), rets0.reshape(-1))]
    for step in range(2):
        X, A, Rt = batches[step]
        for u in range(updates):
            U = step * updates + u
            sl = slice(u * TB, (u + 1) * TB)
            d, _ = O.loss_and_gradients_mt(spec_o, hp, versions[grad_version(U, NT)], X[sl], A[sl], Rt[sl])
            nt, g, ok = O.rmsprop_update(hp, versions[U], g, d)
            assert ok
            versions.append(nt)
    th_o = versions[-1]
    move = np.max(np.abs(th_o - th))
    err = np.max(np.abs(th_dev.astype(np.float64) - th_o))
    gerr = np.max(np.abs(g_dev.astype(np.float64) - g)) / np.max(np.abs(g))
    print(f"theta after 32 updates: max |dev - oracle| {err:.3e}, movement {move:.3e} (ratio {err / move:.2e}); "
          f"g rel {gerr:.2e}")
    assert err <= 1e-5 and err <= 1e-3 * move, (err, move)
    assert gerr <= 2e-4, gerr
