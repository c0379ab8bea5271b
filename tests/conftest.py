import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
ORACLE_DIR = os.path.join(ROOT, "oracle")
if ORACLE_DIR not in sys.path:
    sys.path.insert(0, ORACLE_DIR)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")
    # build the checker and the product if this checkout has not been built yet
    # (the GPU box receives the prebuilt .so files with the snapshot)
    if not os.path.exists(os.path.join(ORACLE_DIR, "libga3c_oracle.so")):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_1611_06256_b200", "libga3c_b200.so")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_1611_06256_b200")],
                       check=True)


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz")))

    return load
