"""bench.py's N > 1 path (torchrun, one process per rank, the fused NVLink
data-parallel update wired through CUDA IPC, barriers and max-over-ranks
timing, one JSON line from rank 0) run as two ranks on the one GPU of the
test box (GA3C_BENCH_ONE_GPU: both ranks on cuda:0, gloo for the
host-side collectives; NCCL refuses two ranks on one device).  The fused
update's own self-check (bitwise against a rank-order sum, dp.py) must pass
-- no fallback -- and the line must report two GPUs and weak scaling."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_fused_update():
    env = dict(os.environ, GA3C_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29583", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "8", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-loop", "--no-large"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["dp_update"] == "fused" and d.get("dp_fallback") is None, (d["config"], d.get("dp_fallback"))
    assert d["config"]["global_train_batch"] == 2 * d["config"]["min_train_batch"]
