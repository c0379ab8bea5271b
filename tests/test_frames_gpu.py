"""Device frame-stack store (include/ga3c.h ga3c_frames_*, SURVEY.md §8f row
1): agents push only their newest frame; the stacked state must equal the
one the host would build (4 frames, oldest first, an episode start repeats
the frame), and predicting / training from the store must give exactly what
ga3c_forward_u8 / ga3c_loss_grad_segments_u8 give on those host states."""
import numpy as np
import pytest

import pyoracle as O

pytestmark = pytest.mark.gpu

H, W = 84, 84


def setup(n_agents=6, history=7, max_batch=64):
    import ctypes as C
    from paper_1611_06256_b200 import _abi
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(O.dnn_a()), C.sizeof(spec))
    m = _abi.Model(spec, _abi.default_hyper())
    th = np.zeros(m.P, np.float32)
    _abi.check(_abi.lib.ga3c_init_params(spec, 3, None, th.ctypes.data))
    m.load(th)
    ctx = _abi.Context(m, max_batch)
    fr = _abi.Frames(m, n_agents, history)
    return _abi, m, ctx, fr


def host_stack(prev, f, reset):
    if prev is None or reset:
        return np.repeat(f[:, :, None], 4, axis=2)
    return np.concatenate([prev[:, :, 1:], f[:, :, None]], axis=2)


def test_push_builds_stacks_and_predicts_like_forward_u8():
    _abi, m, ctx, fr = setup()
    rng = np.random.default_rng(0)
    stacks = {}
    for step in range(9):
        agents = rng.permutation(6)[: rng.integers(1, 7)].astype(np.int32)
        new = rng.integers(0, 256, (len(agents), H, W), dtype=np.uint8)
        resets = (rng.random(len(agents)) < 0.2).astype(np.uint8)
        pi, v, slots, _ = _abi.predict_frames(ctx, fr, new.reshape(len(agents), -1), agents, resets)
        states = []
        for i, a in enumerate(agents):
            stacks[a] = host_stack(stacks.get(a), new[i], resets[i])
            states.append(stacks[a].reshape(-1))
            assert np.array_equal(fr.read(int(a), int(slots[i])), stacks[a].reshape(-1))
        pi2, v2 = ctx.forward(np.stack(states))[:2]
        assert np.array_equal(pi, pi2) and np.array_equal(v, v2)


def test_train_from_store_matches_host_states_bitwise():
    _abi, m, ctx, fr = setup(n_agents=4, history=7)
    rng = np.random.default_rng(1)
    T = 5
    slots = np.zeros((4, T), np.int32)
    states = np.zeros((4, T, H * W * 4), np.uint8)
    stacks = {}
    for t in range(T):
        new = rng.integers(0, 256, (4, H, W), dtype=np.uint8)
        _, _, sl, _ = _abi.predict_frames(ctx, fr, new.reshape(4, -1), np.arange(4, dtype=np.int32))
        slots[:, t] = sl
        for a in range(4):
            stacks[a] = host_stack(stacks.get(a), new[a], False)
            states[a, t] = stacks[a].reshape(-1)
    agents = np.repeat(np.arange(4, dtype=np.int32), T)
    acts = rng.integers(0, 6, 4 * T).astype(np.int32)
    rew = rng.standard_normal(4 * T)
    off = np.arange(0, 4 * T + 1, T, dtype=np.int32)
    term = np.array([0, 1, 0, 0], np.uint8)
    boot = rng.standard_normal(4)
    sc1, r1 = _abi.train_frames(ctx, fr, agents, slots.reshape(-1), acts, rew, off, term, boot, 0.99)
    g1 = ctx.read_grad()[0].copy()
    sc2, r2 = ctx.loss_grad_segments(states.reshape(4 * T, -1), acts, rew, off, term, boot, 0.99)[:2]
    g2 = ctx.read_grad()[0]
    assert np.array_equal(r1, r2) and np.array_equal(sc1, sc2) and np.array_equal(g1, g2)


def test_frames_validation():
    _abi, m, ctx, fr = setup(n_agents=2, history=3)
    with pytest.raises(ValueError):
        _abi.predict_frames(ctx, fr, np.zeros((1, H * W), np.uint8), np.array([5], np.int32))
    with pytest.raises(ValueError):
        _abi.train_frames(ctx, fr, [0], [9], [0], [0.0], [0, 1], [1], [0.0], 0.99)


def test_ring_apply_matches_published_apply():
    """ga3c_model_ring + ga3c_apply_rmsprop_slots_dev (the multi-trainer
    device loop) apply the same RMSProp step as ga3c_apply_rmsprop."""
    _abi, m1, ctx1, _ = setup()
    _, m2, ctx2, _ = setup()
    rng = np.random.default_rng(3)
    states = rng.integers(0, 256, (8, H * W * 4), dtype=np.uint8)
    acts = rng.integers(0, 6, 8).astype(np.int32)
    rets = rng.standard_normal(8)
    d, _ = ctx1.loss_grad(states, acts, rets)
    ring = m1.ring(2)
    ctx1.apply_slots_dev(ctx1, ring[0], ring[1])
    ctx1.sync()
    pi1, v1, _ = ctx1.forward(states, slot=ring[1])
    ctx2.apply_rmsprop(d)
    pi2, v2, _ = ctx2.forward(states)
    assert np.array_equal(pi1, pi2) and np.array_equal(v1, v2)


def test_ring_apply_rejected_step_leaves_source_in_destination():
    """A non-finite gradient rejects the step (nnet.cpp:299-301); out of place
    the destination slot must then hold the unchanged source parameters."""
    import torch
    _abi, m1, ctx1, _ = setup()
    rng = np.random.default_rng(4)
    states = rng.integers(0, 256, (8, H * W * 4), dtype=np.uint8)
    acts = rng.integers(0, 6, 8).astype(np.int32)
    rets = np.full(8, 3e38)  # finite returns whose gradient overflows fp32
    d, _ = ctx1.loss_grad(states, acts, rets)
    assert not np.all(np.isfinite(d))
    ring = m1.ring(3)

    def theta(slot):
        class _V:
            __cuda_array_interface__ = {"shape": (m1.P,), "typestr": "<f4", "version": 3, "strides": None,
                                        "data": (_abi.slot_theta_ptr(m1, slot), False)}
        return torch.as_tensor(_V(), device="cuda").cpu().numpy().copy()

    # make the destination differ from the source first: a valid step into it
    ctx2 = _abi.Context(m1, 8)
    ctx2.loss_grad(states, acts, rng.standard_normal(8))
    ctx2.apply_slots_dev(ctx2, ring[0], ring[2])
    ctx2.sync()
    assert not np.array_equal(theta(ring[2]), theta(ring[1]))
    ctx1.apply_slots_dev(ctx1, ring[1], ring[2])  # rejected: ctx1's gradient is non-finite
    ctx1.sync()
    assert np.array_equal(theta(ring[2]), theta(ring[1]))


def test_async_predict_matches_sync_and_guards_the_stage():
    """ga3c_predict_frames64_async + _collect64 give the bits of
    ga3c_predict_frames64 on an identical store; a second submit, a host
    training call, or a collect with nothing pending are rejected."""
    _abi, m, ctx, fr = setup(n_agents=5, history=4)
    fr2 = _abi.Frames(m, 5, 4)
    ctx2 = _abi.Context(m, 64)
    rng = np.random.default_rng(3)
    agents = np.arange(5, dtype=np.int32)
    for step in range(3):
        new = rng.integers(0, 256, (5, H * W), dtype=np.uint8)
        pi, v, sl, ver = _abi.predict_frames(ctx, fr, new, agents, fp64=True)
        sl2 = _abi.predict_frames_async(ctx2, fr2, new, agents)
        with pytest.raises(ValueError):
            _abi.predict_frames_async(ctx2, fr2, new, agents)  # one in flight per context
        with pytest.raises(ValueError):
            ctx2.loss_grad_segments(np.zeros((5, H * W * 4), np.uint8), np.zeros(5, np.int32), np.zeros(5),
                                    [0, 5], [1], [0.0], 0.99)  # the stage is busy
        pi2, v2, ver2 = _abi.predict_collect(ctx2)
        assert np.array_equal(sl, sl2) and np.array_equal(pi, pi2) and np.array_equal(v, v2) and ver == ver2
    ctx2._pending = (1,)
    with pytest.raises(ValueError):
        _abi.predict_collect(ctx2)


def test_device_sampled_actions_match_host_sample_index():
    """ga3c_predict_frames_act64_async draws each agent's action on the
    device from its uniform: the same action the reference's host-side
    qac::sample_index (util.hpp:46-54, restated in oracle/pyoracle.py)
    draws from the returned fp64 pi, including uniforms placed exactly on
    and just beside a cumulative-probability boundary and u -> 1 (the
    last action).  The pi / V / state slots are those of the host-sampling
    call, and ga3c_predict_collect64 also collects such a prediction."""
    _abi, m, ctx, fr = setup(n_agents=7, history=4)
    fr2 = _abi.Frames(m, 7, 4)
    ctx2 = _abi.Context(m, 64)
    rng = np.random.default_rng(11)
    agents = np.arange(7, dtype=np.int32)
    margins = []
    for step in range(4):
        new = rng.integers(0, 256, (7, H * W), dtype=np.uint8)
        pi, v, sl, ver = _abi.predict_frames(ctx, fr, new, agents, fp64=True)
        cdf = np.cumsum(pi, 1)  # left-to-right fp64, as the reference accumulates
        u = rng.random(7)
        u[0] = cdf[0, 2]  # exactly on a boundary: not below it, so the next action
        u[1] = np.nextafter(cdf[1, 0], 0.0)  # just below: action 0
        u[2] = 1.0 - 1e-17  # rounds to 1.0 in fp64: past every cumulative sum
        u[3] = 0.0
        if step < 3:
            sl2 = _abi.predict_frames_act_async(ctx2, fr2, new, agents, u)
            a2, v2, pi2, ver2 = _abi.predict_collect_act(ctx2, want_pi=True)
            assert np.array_equal(pi, pi2)
        else:
            sl2 = _abi.predict_frames_act_async(ctx2, fr2, new, agents, u)
            pi2, v2, ver2 = _abi.predict_collect(ctx2)
            assert np.array_equal(pi, pi2)
            continue
        want = np.array([O.sample_index(list(pi[i]), float(u[i])) for i in range(7)], np.int32)
        assert np.array_equal(a2, want), (a2, want)
        assert np.array_equal(sl, sl2) and np.array_equal(v, v2) and ver == ver2
        margins.append(float(np.min(np.abs(cdf - u[:, None]))))
    assert margins[0] == 0.0  # the on-boundary draw was exercised
    with pytest.raises(ValueError):
        _abi.predict_frames_act_async(ctx2, fr2, new, agents, u[:3])  # one uniform per agent


def test_graph_replayed_training_trajectory_matches_eager_bitwise():
    """ga3c_train_frames replays a captured graph per (snapshot slot, shape):
    eight train + apply rounds (the latest slot moves every round, so graphs
    are captured and then replayed) give the same parameters, bit for bit,
    as the same rounds through ga3c_loss_grad_segments_u8 on host states
    (eager launches) on a second model."""
    import ctypes as C
    _abi, m, ctx, fr = setup(n_agents=4, history=16)
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(O.dnn_a()), C.sizeof(spec))
    m2 = _abi.Model(spec, _abi.default_hyper())
    m2.load(m.read()[0])
    c2 = _abi.Context(m2, 64)
    rng = np.random.default_rng(5)
    T = 2
    stacks = {}
    agents = np.arange(4, dtype=np.int32)
    for rnd in range(8):
        slots = np.zeros((4, T), np.int32)
        states = np.zeros((4, T, H * W * 4), np.uint8)
        for t in range(T):
            new = rng.integers(0, 256, (4, H, W), dtype=np.uint8)
            _, _, sl, _ = _abi.predict_frames(ctx, fr, new.reshape(4, -1), agents)
            slots[:, t] = sl
            for a in range(4):
                stacks[a] = host_stack(stacks.get(a), new[a], False)
                states[a, t] = stacks[a].reshape(-1)
        acts = rng.integers(0, 6, 4 * T).astype(np.int32)
        rew = rng.standard_normal(4 * T)
        off = np.arange(0, 4 * T + 1, T, dtype=np.int32)
        term = np.zeros(4, np.uint8)
        boot = rng.standard_normal(4)
        _abi.train_frames(ctx, fr, np.repeat(agents, T), slots.reshape(-1), acts, rew, off, term, boot, 0.99)
        assert ctx.apply_rmsprop()[0]
        c2.loss_grad_segments(states.reshape(4 * T, -1), acts, rew, off, term, boot, 0.99)
        assert c2.apply_rmsprop()[0]
        assert np.array_equal(m.read()[0], m2.read()[0]), rnd


def test_graph_replayed_async_predictions_follow_the_snapshot_bitwise():
    """The asynchronous calls replay a graph captured per (snapshot slot, n,
    outputs, store): across training rounds that move the latest slot (new
    keys, then replays of old ones as the ring wraps), two batch sizes, both
    output kinds and an SM-budget change (which drops the context's graphs),
    every prediction equals the eager synchronous ga3c_predict_frames64 on an
    identical store bit for bit, including the device-drawn actions."""
    _abi, m, ctx, fr = setup(n_agents=6, history=8)
    fr2 = _abi.Frames(m, 6, 8)
    ctx2 = _abi.Context(m, 64)
    rng = np.random.default_rng(21)
    agents = np.arange(6, dtype=np.int32)
    versions = set()
    for rnd in range(10):
        if rnd == 6:  # both: the split plans (and so the bits) follow the budget
            ctx.set_sm_budget(40)
            ctx2.set_sm_budget(40)
        sub = agents if rnd % 3 else agents[:4]  # two batch shapes
        slots = []
        for t in range(2):
            new = rng.integers(0, 256, (len(sub), H * W), dtype=np.uint8)
            pi, v, sl, ver = _abi.predict_frames(ctx, fr, new, sub, fp64=True)
            u = rng.random(len(sub))
            if (rnd + t) % 2:
                sl2 = _abi.predict_frames_act_async(ctx2, fr2, new, sub, u)
                a2, v2, pi2, ver2 = _abi.predict_collect_act(ctx2, want_pi=True)
                want = np.array([O.sample_index(list(pi[i]), float(u[i])) for i in range(len(sub))], np.int32)
                assert np.array_equal(a2, want), (rnd, t)
            else:
                sl2 = _abi.predict_frames_async(ctx2, fr2, new, sub)
                pi2, v2, ver2 = _abi.predict_collect(ctx2)
            assert np.array_equal(sl, sl2) and ver == ver2, (rnd, t)
            assert np.array_equal(pi, pi2) and np.array_equal(v, v2), (rnd, t)
            versions.add(ver)
            slots.append(sl)
        n = len(sub)
        acts = rng.integers(0, 6, 2 * n).astype(np.int32)
        off = np.arange(0, 2 * n + 1, 2, dtype=np.int32)
        _abi.train_frames(ctx, fr, np.repeat(sub, 2), np.stack(slots, 1).reshape(-1), acts, rng.standard_normal(2 * n),
                          off, np.zeros(n, np.uint8), rng.standard_normal(n), 0.99)
        assert ctx.apply_rmsprop()[0]
    assert len(versions) == 10
