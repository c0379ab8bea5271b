#!/usr/bin/env python
"""Per-kernel-class roofline table from a bench.py JSON line (SURVEY.md §8d:
achieved / min(tensor peak, AI x HBM) per kernel).

Times are bench.py's `kernel_breakdown_ms_per_step` (per class and layer,
CUDA events around every launch in an eager step); work is algorithmic:
FLOPs from bench.work_per_step, bytes = each operand and result read or
written once (activations fp32, frames u8, RMSProp 20 B/param).  Run bench
with --trainers 1 for a clean serial breakdown.

  python tools/roofline_table.py bench.json [--md out.md]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def class_bytes(net, agents, tmax, tb):
    layers, _ = bench.layer_geometry(net)
    n_fwd = 2 * agents * tmax   # predictor + trainer recompute
    n_tr = agents * tmax
    updates = n_tr // tb
    l_fwd = tmax + updates      # forward launches per step (predictor batches + trainer recomputes)
    out = {}
    h, w, c = bench.FRAME
    in_b = h * w * c  # u8 state
    for li, l in enumerate(layers):
        o = l["N"] * l["P"] * 4
        wb = l["params"] * 4
        key = "conv_fwd" if l["kind"] == "conv" else "fc_fwd"
        out[(key, li)] = float(in_b + o) * n_fwd + wb * l_fwd
        out[("wgrad", li)] = float(in_b + o) * n_tr + wb * updates
        if li > 0:
            out[("dgrad", li)] = float(o + 2 * in_b) * n_tr + wb * updates
        in_b = o
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("json")
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    d = json.loads(open(a.json).read().strip().splitlines()[-1])
    cfg = d["config"]
    net, NA, T, TB = cfg["net"], cfg["agents_per_gpu"], cfg["t_max"], cfg["min_train_batch"]
    flops = bench.work_per_step(net, NA, T, TB)
    byts = class_bytes(net, NA, T, TB)
    P = bench.param_count(net)
    byts[("rmsprop", -1)] = 20.0 * P * (NA * T // TB)
    hbm, bf16, _, src = bench.measured_peaks()
    ridge = bf16 * 1e3 / hbm
    bd = d["kernel_breakdown_ms_per_step"]
    rows = []
    for (cls, li), f in sorted(flops.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        key = f"{cls}[{li}]" if li >= 0 else cls
        ms = bd.get(key)
        if not ms:
            continue
        b = byts.get((cls, li))
        t = ms / 1e3
        if cls == "rmsprop":
            ach, bound, unit, fr = b / t / 1e9, hbm, "GB/s", b / t / 1e9 / hbm
            ai = None
        else:
            ai = f / b if b else None
            bound_tf = min(bf16, ai * hbm / 1e3) if ai else bf16
            ach = f / t / 1e12
            fr = ach / bound_tf
            bound, unit = bound_tf, "TFLOP/s"
        rows.append((key, ms, ai, ach, unit, bound, fr))
    lines = [f"# Per-kernel roofline ({net}, {d['config'].get('trainers_in_flight')} trainer(s) in flight), "
             f"peaks {src}: bf16 {bf16:.0f} TFLOP/s, HBM {hbm:.0f} GB/s, ridge {ridge:.0f} FLOP/B", "",
             "| kernel class | ms/step | FLOP/B | achieved | bound (min(TC, AI x HBM)) | frac |",
             "|---|---|---|---|---|---|"]
    for key, ms, ai, ach, unit, bound, fr in rows:
        lines.append(f"| {key} | {ms:.4f} | {'' if ai is None else f'{ai:.0f}'} | {ach:.1f} {unit} | "
                     f"{bound:.0f} {unit} | {fr:.4f} |")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if a.md:
        open(a.md, "w").write(txt)


if __name__ == "__main__":
    main()
