"""The reference's own engine and Python module running on libga3c_b200.

oracle/Makefile target `dropin` compiles the reference's UNMODIFIED engine
sources (/root/reference/proj/src/{pipeline,reference,envs,metrics,annealer}.cpp
and bindings/qac_module.cpp) with include/ ahead of the reference's include/,
so `#include "qac/nnet.hpp"` / `"qac/returns.hpp"` resolve to the drop-in
shims (include/qac/) and every nnet:: / returns:: call runs on the B200
library.  The same engine is also linked against the reference's own CPU
nnet.cpp / returns.cpp (test_dropin_cpu): the checker.  The binaries are built
in this container (where /root/reference exists) and travel to the GPU box
under oracle/_ref/ like the other checker builds.

CPU tests: the checker build passes the restated reference pipeline tests,
and the B200 build links the product library.  GPU tests: the same tests on
the B200 build, the reference's train_sync trajectory on the device against
the CPU reference, and the reference's Python smoke tests
(tests/python/test_smoke.py:8-129) through its own pybind module.
"""
import importlib.util
import math
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROP = os.path.join(ROOT, "oracle", "_ref", "dropin")
B200 = os.path.join(DROP, "test_dropin_b200")
CPU = os.path.join(DROP, "test_dropin_cpu")

needs_build = pytest.mark.skipif(not os.path.exists(B200) or not os.path.exists(CPU),
                                 reason="drop-in builds missing (make -C oracle dropin, needs /root/reference)")


def _run(exe, *args, timeout=600):
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout)


def _read_traj(path):
    with open(path, "rb") as f:
        n, P = struct.unpack("<qq", f.read(16))
        th = np.frombuffer(f.read(8 * n * P), np.float64).reshape(n, P)
        (k,) = struct.unpack("<q", f.read(8))
        scores = np.frombuffer(f.read(8 * k), np.float64)
    return th, scores


@needs_build
def test_checker_build_passes_reference_pipeline_tests():
    r = _run(CPU, "run")
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


@needs_build
def test_b200_build_links_the_product_library():
    out = subprocess.run(["ldd", B200], capture_output=True, text=True).stdout
    line = [ln for ln in out.splitlines() if "libga3c_b200.so" in ln]
    assert line and "not found" not in line[0], out
    # the engine's math symbols come from the adapter, not from a CPU nnet.o
    syms = subprocess.run(["nm", "-C", "--defined-only", B200], capture_output=True, text=True).stdout
    assert "qac::nnet::forward" not in syms and "qac_b200::nnet::forward" not in syms


@pytest.mark.gpu
@needs_build
def test_reference_engine_on_b200_passes_its_pipeline_tests():
    """test_pipeline.cpp:45-320 through the reference's own pipeline.cpp /
    reference.cpp on the device: one-forward predictor batches, the
    pred_batch_max cap, immutable snapshots, lockstep == train_sync bitwise,
    conservation, coalescing, stop conditions, annealing, validation."""
    r = _run(B200, "run")
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


@pytest.mark.gpu
@needs_build
def test_train_sync_trajectory_matches_cpu_reference(tmp_path):
    """reference::train_sync (reference.cpp:25-157) on catch_grid(4), {16}
    trunk: the device trajectory against the reference's fp64 CPU run of the
    same unmodified engine.  Actions are sampled from the device's fp64
    softmax, so both runs play the same episodes unless a uniform draw falls
    within ~1e-7 of a CDF boundary (then the check below fails loudly)."""
    updates = 60
    for seed in (7, 19):
        a, b = tmp_path / f"g{seed}.bin", tmp_path / f"c{seed}.bin"
        assert _run(B200, "traj", str(seed), str(updates), str(a)).returncode == 0
        assert _run(CPU, "traj", str(seed), str(updates), str(b)).returncode == 0
        tg, sg = _read_traj(a)
        tc, sc = _read_traj(b)
        assert tg.shape == tc.shape == (updates, tg.shape[1])
        assert np.array_equal(sg, sc), "episode scores differ: a sampled action flipped"
        err = np.abs(tg - tc).max(1) / np.abs(tc).max(1)
        print(f"seed {seed}: max rel theta deviation per update: first {err[0]:.2e}, max {err.max():.2e}")
        # fp32 device arithmetic vs fp64: ~1e-7 per update, RMSProp-normalised
        # steps of eta = 3e-4 keep the drift linear in the update count
        assert err.max() < 1e-4, err


def _qac():
    path = [os.path.join(DROP, "b200", f) for f in os.listdir(os.path.join(DROP, "b200")) if f.startswith("_qac")]
    spec = importlib.util.spec_from_file_location("_qac", path[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.gpu
@needs_build
def test_reference_python_module_on_b200(tmp_path):
    """The reference's Python smoke tests (tests/python/test_smoke.py:8-129)
    restated against its own pybind module (bindings/qac_module.cpp) built
    over the drop-in headers."""
    qac = _qac()
    # :8-19 returns, bitwise
    got = qac.compute_returns([1.0, -0.5, 2.0], False, 0.25, 0.9)
    r2 = 2.0 + 0.9 * 0.25
    r1 = -0.5 + 0.9 * r2
    assert got == [1.0 + 0.9 * r1, r1, r2]
    assert qac.compute_returns([1.0], True, 123.0, 0.5) == [1.0]
    with pytest.raises(ValueError):
        qac.compute_returns([], False, 0.0, 0.9)
    # :22-31 forward gives distributions (fp64 softmax across the ABI)
    spec = qac.NetworkSpec(4, [8], 3)
    assert qac.param_count(spec) == 76
    model = qac.init_model(spec, 7)
    out = qac.forward(model, spec, [[0.1, -0.2, 0.3, 0.9], [1.0, 1.0, 1.0, 1.0]])
    assert len(out.policies) == 2 and len(out.values) == 2
    for pi in out.policies:
        assert len(pi) == 3 and all(p >= 0.0 for p in pi)
        assert math.isclose(sum(pi), 1.0, rel_tol=0, abs_tol=1e-12)
    # :34-47 a gradient step moves the parameters
    hyper = qac.Hyperparams()
    model = qac.init_model(spec, 11)
    grads = qac.loss_and_gradients(model, spec, hyper, [[0.5, 0.0, -0.5, 1.0]], [2], [1.5])
    assert all(math.isfinite(d) for d in grads.dtheta)
    step = qac.rmsprop_update(model, qac.init_rms(spec), grads, hyper)
    assert step.applied and step.model.version == 1 and step.model.theta != model.theta
    # :68-91 serial and lock-step pipeline runs agree bit for bit
    env = qac.catch_grid(4)
    net = qac.net_for_env(env, [12])
    sc = qac.SyncConfig()
    sc.env, sc.net, sc.max_updates, sc.seed, sc.capture_trajectory = env, net, 60, 5, True
    serial = qac.train_sync(sc)
    assert serial.total_updates == 60 and serial.mean_lag == 0.0
    opt = qac.PipelineOptions()
    opt.env, opt.net = env, net
    opt.knobs.n_agents = opt.knobs.n_predictors = opt.knobs.n_trainers = 1
    opt.stop.max_updates, opt.seed = 60, 5
    opt.sync_after_submit = opt.capture_trajectory = True
    piped = qac.run(opt)
    assert piped.theta_trajectory == serial.theta_trajectory
    assert piped.final_model.theta == serial.final_model.theta
    # :94-116 every experience is accounted for; frames reconstruct the updates
    opt = qac.PipelineOptions()
    opt.env = qac.bandit()
    opt.net = qac.net_for_env(opt.env, [8])
    opt.knobs.n_agents = 2
    opt.stop.max_updates, opt.seed = 150, 2
    opt.metrics_interval_s = 0.05
    opt.metrics_out = str(tmp_path / "frames.csv")
    rep = qac.run(opt)
    assert rep.total_updates == 150
    assert rep.experiences_produced == rep.experiences_trained + rep.experiences_left_queued + rep.experiences_dropped
    frames = qac.read_frames(rep.metrics_path)
    assert frames and frames[-1].updates_total == 150
    recovered, prev = 0, 0.0
    for f in frames:
        recovered += round(f.tps * (f.wall_time_s - prev))
        prev = f.wall_time_s
    assert recovered == 150
