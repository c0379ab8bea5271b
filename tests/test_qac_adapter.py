"""The reference's nnet/returns unit tests (test_nnet.cpp, test_returns.cpp)
restated in C++ against the drop-in headers include/qac/{nnet,returns}.hpp,
which shadow the reference headers of the same names.  Compiling and linking is
checked on CPU; running needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1611_06256_b200")


def _build(out):
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-Wall", "-Wextra", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_qac_adapter.cpp"),
                    "-L", PKG, "-lga3c_b200", "-Wl,-rpath," + PKG, "-o", str(out)], check=True)


def test_adapter_compiles_and_links(tmp_path):
    _build(tmp_path / "t")
    assert (tmp_path / "t").exists()


@pytest.mark.gpu
def test_adapter_reference_unit_tests(tmp_path):
    exe = tmp_path / "t"
    _build(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
