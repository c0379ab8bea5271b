"""Debug helper: per-layer relative gradient error of the CUDA path vs the oracle."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402
from paper_1611_06256_b200 import _abi  # noqa: E402


def slices(spec):
    out = []
    off = 0
    h, w, c = spec.in_h, spec.in_w, spec.in_c
    for i in range(spec.n_conv):
        co, k, s = spec.conv_out[i], spec.conv_k[i], spec.conv_stride[i]
        n = co * k * k * c
        out += [(f"conv{i}.W", off, off + n), (f"conv{i}.b", off + n, off + n + co)]
        off += n + co
        h, w, c = (h - k) // s + 1, (w - k) // s + 1, co
    prev = h * w * c
    for i in range(spec.n_hidden):
        o = spec.hidden[i]
        out += [(f"fc{i}.W", off, off + prev * o), (f"fc{i}.b", off + prev * o, off + prev * o + o)]
        off += prev * o + o
        prev = o
    A = spec.n_actions
    out += [("pi.W", off, off + prev * A), ("pi.b", off + prev * A, off + prev * A + A)]
    off += prev * A + A
    out += [("v.W", off, off + prev), ("v.b", off + prev, off + prev + 1)]
    return out


def main(net="dnn_a", B=1):
    spec_o = O.dnn_a() if net == "dnn_a" else O.dnn_large(int(net[-1]))
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(spec_o), C.sizeof(spec))
    m = _abi.Model(spec, _abi.default_hyper())
    ctx = _abi.Context(m, max(B, 8))
    th = O.init_model(spec_o, 1).astype(np.float32)
    m.load(th)
    fr = O.synthetic_frames(3, B)
    acts, rets = O.synthetic_batch(3, B, 6)
    d, sc = ctx.loss_grad(fr, acts, rets)
    rd, rsc = O.loss_and_gradients(spec_o, O.Hyper(), th.astype(np.float64), O.frames_to_states(fr), acts, rets)
    for name, a, b in slices(spec_o):
        g, r = d[a:b].astype(np.float64), rd[a:b]
        rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
        print(f"{name:8s} n={b-a:8d} rel={rel:.3e} |ref|={np.linalg.norm(r):.3e} |got|={np.linalg.norm(g):.3e}")
    print("scalars", sc, rsc)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "dnn_a", int(sys.argv[2]) if len(sys.argv) > 2 else 1)
