"""bench.py's JSON contract on CPU: the reference arm (the oracle port on the
host cores) runs here, and its line carries the keys the driver reads, with
the same config the GPU arm prints (SM budgets resolved in parse())."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_param_counts_match_the_layouts():
    assert bench.param_count("dnn_a") == 677943
    assert bench.param_count("large1") == 4794503
    assert abs(bench.fwd_flops_per_sample("dnn_a") / 1e6 - 5.934592) < 1e-6


def test_reference_arm_json_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "libga3c_oracle.so")):
        pytest.skip("oracle not built (run __graft_entry__.build())")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    cfg = d["config"]
    assert cfg["net"] == "dnn_a" and cfg["updates_per_step"] == 16 and cfg["params"] == 677943
    # the GPU arm resolves the same automatic budgets and prints the same
    # dict (config_of has no run-specific keys: the L2 note is top-level)
    assert cfg["trainer_sm_budget"] == 111 and cfg["predictor_sm_budget"] == 40
    assert "l2" not in cfg
    # the reference's lag metric (pipeline.cpp:289-291) for the overlapped
    # N_T = 6 step: 16 + 15/2 updates
    assert cfg["mean_policy_lag_updates"] == 23.5 and cfg["gradient_staleness_updates"] == 5
    assert "executed GA3C iterations" in cb["sample"]


def test_algorithmic_bytes_and_issued_work():
    w = bench.work_per_step("dnn_a", 128, 5, 40)
    b = bench.bytes_per_step("dnn_a", 128, 5, 40)
    # every timed class has both its FLOPs and its bytes
    assert set(w) <= set(b) | {k for k in w if k[0] == "rmsprop"}
    assert b[("rmsprop", -1)] == 20.0 * 677943 * 16 == w[("rmsprop", -1)]
    # conv1 weight gradient: u8 frame + fp32 output gradient per sample
    assert b[("wgrad", 0)] == (28224 + 20 * 20 * 16 * 4) * 640 + 4 * (16 * 8 * 8 * 4 + 16) * 16
    assert bench.issued(("wgrad", 0)) == ("tf32", 2.0) and bench.issued(("dgrad", 1)) == ("tf32", 3.0)


def test_reference_arm_under_torchrun_prints_one_line():
    """N > 1: the driver launches the reference arm with torchrun; rank 0
    alone runs the CPU path and prints, the other ranks exit 0."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "libga3c_oracle.so")):
        pytest.skip("oracle not built (run __graft_entry__.build())")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_ncu_traffic_entries_per_net():
    """roofline.traffic comes from profiles/ncu_traffic.json, keyed by net and
    probed kernel class (DRAM read + write bytes of one ncu --set full launch)."""
    d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    for net in ("dnn_a", "large1"):
        e = d[net]["conv_fwd[0]"]
        assert e["bytes_per_launch"] == e["read"] + e["write"] > 0
        assert e["algorithmic_bytes"] > 0 and e["capture"].startswith("profiles/")
        assert os.path.exists(os.path.join(ROOT, e["capture"].split(" ")[0]))
