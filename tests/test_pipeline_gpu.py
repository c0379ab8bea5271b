"""The B200 host engine (csrc/host, C++) through the C ABI: the reference's
pipeline tests (proj/tests/test_pipeline.cpp, test_reference.cpp,
tests/python/test_smoke.py) restated.  Needs a GPU: -m gpu."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def q():
    from paper_1611_06256_b200 import qac
    return qac


def lockstep(env, updates, seed, hidden=(16,)):
    qac = q()
    opt = qac.PipelineOptions(net=qac.net_for_env(env, list(hidden)), env=env)
    opt.knobs = qac.KnobConfig(n_agents=1, n_predictors=1, n_trainers=1, min_train_batch=1)
    opt.stop = qac.StopCondition(max_updates=updates)
    opt.seed = seed
    opt.sync_after_submit = True
    return opt


@pytest.mark.parametrize("seed", [7, 19])
def test_lockstep_pipeline_reproduces_sync_trainer_bitwise(seed):  # test_pipeline.cpp:123-148
    qac = q()
    opt = lockstep(qac.catch_grid(4), 120, seed)
    opt.capture_trajectory = True
    piped = qac.run(opt)
    serial = qac.train_sync(opt)
    assert piped.total_updates == 120 and serial.total_updates == 120
    assert len(piped.theta_trajectory) == 120 and len(serial.theta_trajectory) == 120
    for a, b in zip(piped.theta_trajectory, serial.theta_trajectory):
        assert np.array_equal(a, b)
    assert np.array_equal(piped.final_theta, serial.final_theta)
    assert piped.episode_scores == serial.episode_scores
    assert piped.mean_lag == 0.0


def test_lockstep_frames_dnn_a_bitwise():
    """The same equivalence on pixels through DNN A (tensor-core path)."""
    qac = q()
    env = qac.frame_catch(7, 6)
    opt = lockstep(env, 12, 3)
    opt.net = qac.dnn_a()
    opt.capture_trajectory = True
    a = qac.run(opt)
    b = qac.train_sync(opt)
    for x, y in zip(a.theta_trajectory, b.theta_trajectory):
        assert np.array_equal(x, y)


def test_greedy_lockstep_reproducible():  # test_pipeline.cpp:150-158
    qac = q()
    opt = lockstep(qac.catch_grid(4), 40, 33)
    opt.greedy = True
    a, b = qac.run(opt), qac.run(opt)
    assert np.array_equal(a.final_theta, b.final_theta)
    assert a.total_episodes == b.total_episodes and a.episode_scores == b.episode_scores


def test_every_experience_accounted_for():  # test_pipeline.cpp:160-177
    qac = q()
    env = qac.catch_grid(5)
    opt = qac.PipelineOptions(net=qac.net_for_env(env, [16]), env=env)
    opt.knobs = qac.KnobConfig(n_agents=3, n_predictors=2, n_trainers=2, min_train_batch=8)
    opt.stop = qac.StopCondition(max_updates=60)
    opt.seed = 123
    r = qac.run(opt)
    assert r.total_updates == 60
    assert r.experiences_produced == r.experiences_trained + r.experiences_left_queued + r.experiences_dropped
    assert r.experiences_trained >= 60 * 8
    assert r.total_episodes == len(r.episode_scores)


def test_trainers_coalesce_to_batch_floor():  # test_pipeline.cpp:179-196
    qac = q()
    env = qac.bandit()
    opt = qac.PipelineOptions(net=qac.net_for_env(env, [8]), env=env)
    opt.knobs = qac.KnobConfig(n_agents=2, n_predictors=1, n_trainers=1, min_train_batch=7)
    opt.stop = qac.StopCondition(max_updates=25)
    opt.seed = 5
    r = qac.run(opt)
    assert r.total_updates == 25 and r.experiences_trained == 25 * 7
    assert r.experiences_produced == r.experiences_trained + r.experiences_left_queued + r.experiences_dropped


def test_free_running_pipeline_records_staleness():  # test_pipeline.cpp:198-219
    qac = q()
    env = qac.catch_grid(5)
    opt = qac.PipelineOptions(net=qac.net_for_env(env, [16]), env=env)
    opt.knobs = qac.KnobConfig(n_agents=4, n_predictors=1, n_trainers=1, min_train_batch=1)
    opt.stop = qac.StopCondition(max_updates=300)
    opt.seed = 99
    r = qac.run(opt)
    assert r.total_updates == 300 and r.mean_lag >= 0.0 and math.isfinite(r.mean_lag)
    assert r.final_knobs.n_agents == 4


def test_stop_conditions_and_learning():  # test_pipeline.cpp:221-244
    qac = q()
    env = qac.bandit(2, 2)
    opt = qac.PipelineOptions(net=qac.net_for_env(env, [8]), env=env)
    opt.knobs = qac.KnobConfig(n_agents=1, n_predictors=1, n_trainers=1)
    opt.stop = qac.StopCondition(max_seconds=0.3)
    opt.seed = 3
    r = qac.run(opt)
    assert 0.3 <= r.wall_time_s < 30 and r.total_updates > 0
    opt.stop = qac.StopCondition(target_score=0.9)
    opt.hyper = qac.Hyperparams(eta=0.01)
    r2 = qac.run(opt)
    assert r2.final_rolling_score >= 0.9 and r2.total_episodes >= 30


def test_annealing_stays_within_limits():  # test_pipeline.cpp:246-276
    qac = q()
    env = qac.bandit()
    opt = qac.PipelineOptions(net=qac.net_for_env(env, [8]), env=env)
    opt.knobs = qac.KnobConfig(n_agents=2, n_predictors=1, n_trainers=1)
    opt.anneal = True
    opt.epoch_s = 0.2
    opt.limits = (4, 3, 3)
    opt.stop = qac.StopCondition(max_seconds=2.0)
    opt.seed = 17
    r = qac.run(opt)
    assert len(r.anneal_history) >= 2
    for h in r.anneal_history:
        k = h["knobs"]
        assert 1 <= k.n_agents <= 4 and 1 <= k.n_predictors <= 3 and 1 <= k.n_trainers <= 3
        assert h["measured_tps"] >= 0
    assert r.final_knobs.min_train_batch == 1 and r.final_knobs.pred_batch_max == 32


def test_pipeline_validation():  # test_pipeline.cpp:278-314
    qac = q()
    good = lockstep(qac.bandit(), 5, 1)
    bad = lockstep(qac.bandit(), 5, 1)
    bad.stop = qac.StopCondition()
    with pytest.raises(ValueError):
        qac.run(bad)
    bad = lockstep(qac.bandit(), 5, 1)
    bad.knobs.n_agents = 2
    with pytest.raises(ValueError):
        qac.run(bad)
    bad = lockstep(qac.bandit(), 5, 1)
    bad.net = qac.NetworkSpec(5, [16], 4)
    with pytest.raises(ValueError):
        qac.run(bad)
    bad = lockstep(qac.bandit(), 5, 1)
    bad.knobs.n_predictors = 0
    with pytest.raises(ValueError):
        qac.run(bad)
    assert qac.run(good).total_updates == 5


def test_frame_catch_dnn_a_free_running():
    """DNN A on pixels with several agents / predictors / trainers."""
    qac = q()
    env = qac.frame_catch(7, 6)
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=env)
    opt.knobs = qac.KnobConfig(n_agents=16, n_predictors=2, n_trainers=2, pred_batch_max=16, min_train_batch=20)
    opt.stop = qac.StopCondition(max_updates=50)
    r = qac.run(opt)
    assert r.total_updates == 50 and r.experiences_trained >= 50 * 20
    assert r.total_predictions >= r.experiences_produced
    assert np.all(np.isfinite(r.final_theta))


# ------------------------------------------------ device frame store mode
def test_lockstep_device_frames_equals_whole_states_bitwise():
    """device_frames: agents send only their newest 84x84 frame, the stacks
    are built on the GPU (ga3c_predict_frames64) and training gathers them
    there (ga3c_train_frames).  FrameCatch's host stack and the device stack
    hold the same bytes, so the lock-step run must reproduce train_sync on
    whole states bit for bit (test_pipeline.cpp:123-148)."""
    qac = q()
    env = qac.frame_catch(7, 6)
    opt = lockstep(env, 24, 5)
    opt.net = qac.dnn_a()
    opt.capture_trajectory = True
    opt.device_frames = True
    a = qac.run(opt)
    opt.device_frames = False
    b = qac.train_sync(opt)
    assert a.total_updates == b.total_updates == 24
    for x, y in zip(a.theta_trajectory, b.theta_trajectory):
        assert np.array_equal(x, y)
    assert a.episode_scores == b.episode_scores


def test_device_frames_free_running_accounting():
    qac = q()
    env = qac.frames(episode_len=16)
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=env, device_frames=True)
    opt.knobs = qac.KnobConfig(n_agents=32, n_predictors=2, n_trainers=2, pred_batch_max=32, min_train_batch=40)
    opt.stop = qac.StopCondition(max_updates=200)
    r = qac.run(opt)
    assert r.total_updates == 200 and r.experiences_trained >= 200 * 40
    assert r.experiences_produced == r.experiences_trained + r.experiences_left_queued + r.experiences_dropped
    assert np.all(np.isfinite(r.final_theta))


def test_device_frames_reject_non_frame_env():
    qac = q()
    env = qac.catch_grid(4)
    opt = lockstep(env, 5, 1)
    opt.device_frames = True
    with pytest.raises(ValueError):
        qac.run(opt)


def test_annealer_moves_batch_knobs_in_a_running_pipeline():
    """BASELINE configs[1]'s dynamic scheduling with the batch-geometry
    extension (annealer.cpp:28-53 widened): over short epochs the
    annealer proposes pred_batch_max / min_train_batch moves, the engine
    restarts the predictor / trainer pools with them and keeps training."""
    qac = q()
    env = qac.frames(episode_len=32)
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=env, device_frames=True)
    opt.knobs = qac.KnobConfig(n_agents=16, n_predictors=1, n_trainers=1, pred_batch_max=16, min_train_batch=20)
    opt.anneal = True
    opt.anneal_batches = True
    opt.epoch_s = 0.15
    opt.limits = (16, 3, 3)
    opt.stop = qac.StopCondition(max_seconds=4.0)
    opt.seed = 29
    r = qac.run(opt)
    hist = r.anneal_history
    assert len(hist) >= 8
    moved = {(h["knobs"].pred_batch_max, h["knobs"].min_train_batch) for h in hist}
    assert len(moved) >= 2, moved  # batch geometry was proposed and run
    for h in hist:
        k = h["knobs"]
        assert 1 <= k.n_agents <= 16 and 1 <= k.n_predictors <= 3 and 1 <= k.n_trainers <= 3
        assert 1 <= k.pred_batch_max <= 1024 and 1 <= k.min_train_batch <= 1024
    assert r.total_updates > 0 and np.all(np.isfinite(r.final_theta))


def test_device_frames_backpressure_single_agent_large_batches():
    """One agent against one trainer with min_train_batch 240 and the 256-slot
    frame-store history: the agent outruns training, finds its next slot
    still holding an untrained state, hands its open batch over and waits
    (pipeline.cpp agent_main), and the run still completes with every
    experience accounted for."""
    qac = q()
    env = qac.frames(episode_len=1000)
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=env, device_frames=True)
    opt.knobs = qac.KnobConfig(n_agents=1, n_predictors=1, n_trainers=2, pred_batch_max=1, min_train_batch=240)
    opt.stop = qac.StopCondition(max_updates=12)
    r = qac.run(opt)
    assert r.total_updates == 12 and r.experiences_trained >= 12 * 240
    assert r.experiences_produced == r.experiences_trained + r.experiences_left_queued + r.experiences_dropped
    assert np.all(np.isfinite(r.final_theta))
