"""Two processes on one GPU exchanging the fused data-parallel update's
buffers through CUDA IPC (tests/dp_ipc_worker.py under torchrun, gloo for the
host-side handle exchange): every rank reads each peer's gradient through the
pointer it opened, then one ga3c_dp_apply runs across the processes and the
resulting theta' is compared bitwise with the rank-order sum + fp32 RMSProp
restatement.  (Kernels of different processes are time-sliced on one GPU,
so the cross-rank barriers complete through preemption rather than true
concurrency; on a multi-GPU box they run concurrently over NVLink.)"""
import json
import re
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_two_process_ipc_fused_update():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "tests", "dp_ipc_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    # the two ranks share one stdout pipe: their lines may interleave
    lines = [json.loads(x) for x in re.findall(r"\{[^{}]*\}", r.stdout)]
    print(lines)
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == 2
    for d in lines:
        assert d["wiring_ok"], d
        assert d["fused_ok"], d
        assert d["theta_bitwise"] and d["g_shard_bitwise"], d
