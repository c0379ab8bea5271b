"""Launch B-sample forwards (and optionally one training step) of a net,
for an ncu launch list.  usage: python tools/fwd_probe.py NET B [train]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
from sweep import spec_of  # noqa: E402
from paper_1611_06256_b200 import _abi  # noqa: E402

net, B = sys.argv[1], int(sys.argv[2])
train = len(sys.argv) > 3
spec = spec_of(_abi, net)
model = _abi.Model(spec, _abi.default_hyper(), device=0)
th = np.zeros(model.P, np.float32)
_abi.check(_abi.lib.ga3c_init_params(spec, 1, None, th.ctypes.data))
model.load(th)
slot, _ = model.acquire()
ctx = _abi.Context(model, B)
fr = torch.randint(0, 256, (B,) + bench.FRAME, dtype=torch.uint8, device="cuda")
act = torch.randint(0, bench.N_ACTIONS, (B,), dtype=torch.int32, device="cuda")
ret = (torch.rand(B, dtype=torch.float64, device="cuda") - 0.5) * 4
for _ in range(3):
    if train:
        ctx.loss_grad_dev(fr.data_ptr(), True, act.data_ptr(), ret.data_ptr(), B, slot)
        ctx.apply_rmsprop_dev()
    else:
        ctx.forward_dev(fr.data_ptr(), B, True, slot=slot)
ctx.sync()
