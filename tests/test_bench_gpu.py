"""The benchmark's device step chains up to 8 GA3C iterations per CUDA graph,
with the update index continuous across them so the first updates of one
iteration overlap the last of the previous one (bench.py `step`).  Every
update reads a fixed parameter version (policy lag N_T - 1), so the
parameters after a run are schedule-independent: the fingerprint must be
bitwise equal for 1, 2, 4 and 8 iterations per graph -- a missing dependency
between the chained iterations would show up here."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _fingerprint(graph_steps, extra=()):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "8", "--warmup", "3", "--no-cpu",
           "--no-e2e", "--no-loop", "--no-graph-warm", "--graph-steps", str(graph_steps), *extra]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])["theta_fingerprint"]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("extra", [(), ("--no-overlap",)])
def test_chained_graph_steps_are_schedule_independent(extra):
    f1 = _fingerprint(1, extra)
    assert f1 is not None
    assert _fingerprint(2, extra) == f1
    assert _fingerprint(4, extra) == f1
    assert _fingerprint(8, extra) == f1
