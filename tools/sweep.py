#!/usr/bin/env python
"""Batch-size sweep (BASELINE.json configs[4]): predictor forward and trainer
step (loss/backward + RMSProp) for B = 1 .. 1024 on DNN A and the large net,
device-resident u8 inputs larger than L2, each point a CUDA graph of R
iterations timed with CUDA events on the context stream.  Prints one JSON
line per point plus a markdown table (-> profiles/).  Needs a GPU.

  python tools/sweep.py [--nets dnn_a,large1] [--max-batch 1024] [--md out.md]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (net table, FLOP accounting, measured peaks)


def spec_of(_abi, net):
    convs, hidden = bench.NETS[net]
    s = _abi.NetSpec()
    s.in_h, s.in_w, s.in_c = bench.FRAME
    s.n_conv = len(convs)
    for i, (co, k, st) in enumerate(convs):
        s.conv_out[i], s.conv_k[i], s.conv_stride[i] = co, k, st
    s.n_hidden = len(hidden)
    for i, h in enumerate(hidden):
        s.hidden[i] = h
    s.n_actions = bench.N_ACTIONS
    return s


def train_flops(net):
    layers, heads = bench.layer_geometry(net)
    f = 0.0
    for li, l in enumerate(layers):
        mac = l["K"] * l["N"] * l["P"]
        f += 2.0 * mac * (2 + (li > 0))
    return f + 3 * 2.0 * heads["K"] * heads["N"]


def issued_ceiling(net, kind, tc):
    """Algorithmic TFLOP/s ceiling at the precisions the kernels issue
    (bench.issued: conv1 forward = 4 exact int8 digit MMAs, the u8-input
    weight gradient 2 tf32 MMAs, every other GEMM 3xTF32) against the
    measured dense peaks (profiles/r2_tc_peaks.json): total FLOPs / sum of
    each GEMM's issued-MMA time.  The heads (SIMT, < 0.1% of the FLOPs) are
    left out."""
    layers, _ = bench.layer_geometry(net)
    peak = {"tf32": tc.get("tf32_tflops", 1117.2), "i8": tc.get("i8_tops", 4595.6)}
    flops = t = 0.0
    passes = [("conv_fwd" if l["kind"] == "conv" else "fc_fwd", li) for li, l in enumerate(layers)]
    if kind == "train":
        passes += [("wgrad", li) for li in range(len(layers))] + [("dgrad", li) for li in range(1, len(layers))]
    for tag, li in passes:
        l = layers[li]
        f = 2.0 * l["K"] * l["N"] * l["P"]
        prec, factor = bench.issued((tag, li))
        flops += f
        t += f * factor / (peak[prec] * 1e12)
    return flops / t / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nets", default="dnn_a,large1")
    ap.add_argument("--max-batch", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    import torch
    from paper_1611_06256_b200 import _abi
    hbm, bf16, _, src = bench.measured_peaks()
    tc = bench.tc_peaks()
    rows = []
    for net in a.nets.split(","):
        spec = spec_of(_abi, net)
        model = _abi.Model(spec, _abi.default_hyper(), device=0)
        th = np.zeros(model.P, np.float32)
        _abi.check(_abi.lib.ga3c_init_params(spec, 1, None, th.ctypes.data))
        model.load(th)
        slot, _ = model.acquire()
        ctx = _abi.Context(model, a.max_batch)
        stream = torch.cuda.ExternalStream(ctx.stream)
        fwd_f = bench.fwd_flops_per_sample(net)
        trn_f = train_flops(net)
        B = 1
        while B <= a.max_batch:
            sets = max(2, int(np.ceil(160e6 / (B * bench.FRAME_BYTES))))
            sets = min(sets, max(2, int(2e9 // (B * bench.FRAME_BYTES))))
            fr = torch.randint(0, 256, (sets, B) + bench.FRAME, dtype=torch.uint8, device="cuda")
            act = torch.randint(0, bench.N_ACTIONS, (B,), dtype=torch.int32, device="cuda")
            ret = (torch.rand(B, dtype=torch.float64, device="cuda") - 0.5) * 4
            torch.cuda.synchronize()
            res = {}
            for kind in ("predict", "train"):
                def it(i):
                    p = fr[i % sets].data_ptr()
                    if kind == "predict":
                        ctx.forward_dev(p, B, True, slot=slot)
                    else:
                        ctx.loss_grad_dev(p, True, act.data_ptr(), ret.data_ptr(), B, slot)
                        ctx.apply_rmsprop_dev()
                for i in range(3):
                    it(i)
                ctx.graph_begin()
                for i in range(a.reps):
                    it(i)
                g = ctx.graph_end()
                ctx.graph_launch(g)
                ctx.sync()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    ctx.graph_launch(g)
                e1.record(stream)
                e1.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (5 * a.reps)
                f = (fwd_f if kind == "predict" else trn_f) * B
                res[kind] = {"us": us, "samples_per_s": B / (us * 1e-6), "tflops": f / (us * 1e-6) / 1e12}
            row = {"net": net, "B": B, **{f"{k}_{m}": v[m] for k, v in res.items() for m in v},
                   "peak_tflops": bf16, "peak_source": src}
            row["predict_frac"] = row["predict_tflops"] / bf16
            row["train_frac"] = row["train_tflops"] / bf16
            for k in ("predict", "train"):
                row[f"{k}_issued_ceiling_tflops"] = issued_ceiling(net, k, tc)
                row[f"{k}_frac_issued"] = row[f"{k}_tflops"] / row[f"{k}_issued_ceiling_tflops"]
            print(json.dumps(row), flush=True)
            rows.append(row)
            del fr
            B *= 2
        ctx.close()
        model.close()
    if a.md:
        with open(a.md, "w") as f:
            f.write(f"# Batch-size sweep (tools/sweep.py), bf16 peak = {bf16} TFLOP/s ({src})\n\n")
            f.write("frac = achieved / bf16 peak; frac_issued = achieved / the ceiling at the precisions the "
                    "kernels issue (3xTF32 GEMMs, exact int8-digit conv1 forward) from the measured tf32 / i8 "
                    f"peaks ({tc.get('tf32_tflops')} / {tc.get('i8_tops')} T/s, profiles/r2_tc_peaks.json)\n\n")
            f.write("| net | B | predict us | predictions/s | TFLOP/s | frac | frac_issued | train us | samples/s | "
                    "TFLOP/s | frac | frac_issued |\n")
            f.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['net']} | {r['B']} | {r['predict_us']:.1f} | {r['predict_samples_per_s']:.0f} | "
                        f"{r['predict_tflops']:.2f} | {r['predict_frac']:.4f} | {r['predict_frac_issued']:.3f} | "
                        f"{r['train_us']:.1f} | {r['train_samples_per_s']:.0f} | {r['train_tflops']:.2f} | "
                        f"{r['train_frac']:.4f} | {r['train_frac_issued']:.3f} |\n")


if __name__ == "__main__":
    main()
