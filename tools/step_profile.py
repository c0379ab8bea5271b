"""Graph-mode cost of the pieces of a GA3C step (diagnostic, not the bench)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1611_06256_b200 import _abi  # noqa: E402


def main(net="dnn_a", tb=40, na=128):
    convs, hidden = bench.NETS[net]
    spec = _abi.NetSpec()
    spec.in_h, spec.in_w, spec.in_c = bench.FRAME
    spec.n_conv = len(convs)
    for i, (co, k, s) in enumerate(convs):
        spec.conv_out[i], spec.conv_k[i], spec.conv_stride[i] = co, k, s
    spec.n_hidden = len(hidden)
    for i, h in enumerate(hidden):
        spec.hidden[i] = h
    spec.n_actions = 6
    m = _abi.Model(spec, _abi.default_hyper())
    ctx = _abi.Context(m, max(na, tb))
    th = np.zeros(m.P, np.float32)
    _abi.lib.ga3c_init_params(spec, 1, None, th.ctypes.data)
    m.load(th)
    slot, _ = m.acquire()
    fr = torch.randint(0, 256, (na * 5, 84, 84, 4), dtype=torch.uint8, device="cuda")
    acts = torch.randint(0, 6, (na * 5,), dtype=torch.int32, device="cuda")
    rets = torch.randn(na * 5, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    FB = bench.FRAME_BYTES

    def timeit(name, fn, reps=50):
        for _ in range(3):
            fn()
        ctx.sync()
        ctx.graph_begin()
        fn()
        g = ctx.graph_end()
        for _ in range(3):
            ctx.graph_launch(g)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ctx.graph_launch(g)
        e1.record(stream)
        e1.synchronize()
        print(f"{name:40s} {e0.elapsed_time(e1) / reps * 1000:9.1f} us")

    timeit("16x forward B=40", lambda: [ctx.forward_dev(fr.data_ptr() + u * tb * FB, tb, True, slot=slot) for u in range(16)])
    timeit("5x forward B=128", lambda: [ctx.forward_dev(fr.data_ptr() + t * na * FB, na, True, slot=slot) for t in range(5)])
    timeit("16x loss_grad B=40", lambda: [ctx.loss_grad_dev(fr.data_ptr() + u * tb * FB, True, acts.data_ptr() + 4 * u * tb,
                                                           rets.data_ptr() + 8 * u * tb, tb, slot) for u in range(16)])
    timeit("16x rmsprop", lambda: [ctx.apply_rmsprop_dev() for _ in range(16)])
    timeit("16x (loss_grad + rmsprop)", lambda: [(ctx.loss_grad_dev(fr.data_ptr() + u * tb * FB, True, acts.data_ptr() + 4 * u * tb,
                                                                     rets.data_ptr() + 8 * u * tb, tb, slot), ctx.apply_rmsprop_dev())
                                                    for u in range(16)])
    n0 = ctx.launches()
    ctx.loss_grad_dev(fr.data_ptr(), True, acts.data_ptr(), rets.data_ptr(), tb, slot)
    print("kernels per loss_grad:", ctx.launches() - n0)
    ctx.sync()
    # per-launch timeline of one eager update queued behind a spin (serial
    # latency view: every launch's start/end relative to the first)
    for rep in range(2):
        ctx.time_kernel("all")
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(4e6))
        ctx.loss_grad_dev(fr.data_ptr(), True, acts.data_ptr(), rets.data_ptr(), tb, slot)
        ctx.apply_rmsprop_dev()
        tl = ctx.timeline()
        ctx.time_kernel("none")
    print("# one eager update (B=%d): start_ms end_ms dur_us stream kernel[layer]" % tb)
    for tag, li, sid, a, b in tl:
        print(f"{a:9.4f} {b:9.4f} {1e3 * (b - a):8.2f}  s{sid}  {tag}[{li}]")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["dnn_a"]))
