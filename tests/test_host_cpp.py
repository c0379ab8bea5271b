"""Runs the CPU unit tests of the C++ host engine (tests/cpp/test_host.cpp):
queues, annealer, environments, sampling.  No GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_cpp_units(tmp_path):
    exe = tmp_path / "test_host"
    host = os.path.join(ROOT, "paper_1611_06256_b200", "csrc", "host")
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I", host, "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_host.cpp"), os.path.join(host, "envs.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
