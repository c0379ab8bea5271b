"""Device-only check of DeviceLoop's version schedule for several N_T: the
concurrent loop (one graph of two chained steps) against a serial replay of
the same schedule on one context (same SM budget, so the same split-K plans
and bitwise the same kernels).  Diagnostic, not a test."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402
from paper_1611_06256_b200 import _abi  # noqa: E402
from paper_1611_06256_b200.loop import DeviceLoop, grad_version  # noqa: E402

NA, T, TB = 128, 5, 40
FB = 84 * 84 * 4


def run(NT, overlap=True, graph=True):
    spec_o = O.dnn_a()
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(spec_o), C.sizeof(spec))
    hyper = _abi.default_hyper()
    model = _abi.Model(spec, hyper)
    ctx = _abi.Context(model, NA)
    th0 = O.init_model(spec_o, O.derive_seed(1, [O.SEED_MODEL_INIT])).astype(np.float32)
    model.load(th0)
    rng = np.random.default_rng(7)
    frames = rng.integers(0, 256, (2, NA, T, 84, 84, 4), dtype=np.uint8)
    uni = rng.random((2, T, NA))
    rewards = rng.random((2, NA, T)) * 2 - 1
    terminal = (rng.random((2, NA)) < T / 64.0).astype(np.uint8)
    dev = lambda a: torch.from_numpy(a).cuda()
    d_frames = dev(frames)
    loop = DeviceLoop(model, ctx, NA, T, TB, NT, d_frames, dev(uni), dev(rewards), dev(terminal),
                      trainer_sms=111, pred_sms=64, overlap=overlap, hyper=hyper)
    if graph:
        graphs, _ = loop.capture(G=2)
        loop.launch(graphs[0])
    else:
        loop.step(0, 0)
        loop.step(1, 1)
    loop.sync()
    torch.cuda.synchronize()
    th_dev, g_dev = model.read_slot(loop.latest_slot())
    acts0 = loop.actions2[0].clone()
    rets0 = loop.rets2[0].clone()
    # serial replay: version v in slot v
    m2 = _abi.Model(spec, hyper)
    m2.load(th0)
    c2 = _abi.Context(m2, NA)
    c2.set_sm_budget(111)
    slots = m2.ring(33)
    zeros_a = torch.zeros((NA, T), dtype=torch.int32, device="cuda")
    zeros_r = torch.zeros((NA, T), dtype=torch.float64, device="cuda")
    upd = NA * T // TB
    for step in range(2):
        fr = d_frames[1].data_ptr() if step == 0 else d_frames[0].data_ptr()
        a = zeros_a if step == 0 else acts0
        r = zeros_r if step == 0 else rets0
        for u in range(upd):
            U = step * upd + u
            c2.loss_grad_dev(fr + u * TB * FB, True, a.data_ptr() + 4 * u * TB, r.data_ptr() + 8 * u * TB, TB,
                             slots[grad_version(U, NT)])
            c2.apply_slots_dev(c2, slots[U], slots[U + 1])
    c2.sync()
    th_s, g_s = m2.read_slot(slots[32])
    d = np.abs(th_dev.astype(np.float64) - th_s)
    print(f"NT={NT} overlap={overlap} graph={graph}: bitwise {np.array_equal(th_dev, th_s)} max|d| {d.max():.3e} "
          f"g bitwise {np.array_equal(g_dev, g_s)}", flush=True)


if __name__ == "__main__":
    for NT in (2, 3, 4, 5):
        run(NT)
    run(4, graph=False)
    run(4, overlap=False)
