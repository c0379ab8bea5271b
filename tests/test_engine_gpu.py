"""The host engine's own predictor_loop (ga3c::host, the reference's
test_pipeline.cpp:45-98 restated on it: one forward for everything queued,
bitwise equal to a direct batched forward; batches capped at
pred_batch_max), its device frame-store mode, and the native trainer pool
(bitwise equal to the same train_frames + apply calls made directly).
tests/cpp/test_engine_gpu.cpp linked against libga3c_b200.so.  -m gpu."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1611_06256_b200")

pytestmark = pytest.mark.gpu


def build(tmp_path):
    exe = tmp_path / "test_engine_gpu"
    host = os.path.join(PKG, "csrc", "host")
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I", host, "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_engine_gpu.cpp"), "-L", PKG, "-lga3c_b200",
                    f"-Wl,-rpath,{PKG}", "-o", str(exe)], check=True)
    return exe


def test_engine_predictor_and_trainer_pool(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout, r.stdout
