"""Worker of tests/test_dp_ipc_gpu.py: one rank of a 2-process data-parallel
group on ONE GPU (torchrun, gloo for the host-side exchange).

It exercises the real multi-process wiring of the fused exchange
(dp.FusedUpdate): every rank's gradient buffers, destination thetas and
signal block are exported as CUDA IPC handles, gathered over the process
group and opened in every peer; then one fused update (ga3c_dp_apply) runs
across the two processes and is compared with its definition -- the
rank-order fp32 sum of both gradients followed by the fp32 RMSProp
restatement (oracle orc_rmsprop_update_f32).  Prints one JSON line."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import torch
    import torch.distributed as dist

    import pyoracle as O
    from paper_1611_06256_b200 import _abi, dp

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    spec_o = O.make_spec((12, 12, 2), [(4, 4, 2)], [16], 3)
    spec = _abi.NetSpec()
    C.memmove(C.byref(spec), C.byref(spec_o), C.sizeof(spec))
    hyper = _abi.default_hyper()
    model = _abi.Model(spec, hyper, device=0)
    th = O.init_model(spec_o, 5).astype(np.float32)
    g0 = np.full(th.size, 1e-4, np.float32)
    model.load(th, g0)
    ring = model.ring(2)
    ctx = _abi.Context(model, 4)
    P = model.P
    out = {"rank": rank}

    def pattern(r):
        i = np.arange(P, dtype=np.int64)
        return ((((i * 7 + r * 13) % 101) - 50).astype(np.float32) * np.float32(1e-3 * (1 + r)))

    gv = dp.grad_view(ctx, P, "cuda:0")
    gv.copy_(torch.from_numpy(pattern(rank)).cuda())
    torch.cuda.synchronize()
    fused = dp.FusedUpdate(model, [ctx], ring, rank, world, ctas=8)

    # 1. wiring: read every peer's gradient through the pointer this process opened
    wiring_ok = True
    for q in range(world):
        ptr = fused.peers["grad"][0][q]

        class _V:
            __cuda_array_interface__ = {"shape": (P,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                        "strides": None}
        got = torch.as_tensor(_V(), device="cuda:0").cpu().numpy()
        wiring_ok &= bool(np.array_equal(got, pattern(q)))
    out["wiring_ok"] = wiring_ok
    dist.barrier()

    # 2. one fused update across the two processes
    try:
        fused.apply(ctx, 0, ring[0], ring[1])
        fused.dp.check()
        out["fused_ok"] = True
    except Exception as e:  # reported, the test decides
        out["fused_ok"] = False
        out["fused_error"] = str(e)[:300]
    dist.barrier()
    if out["fused_ok"]:
        th1, g1 = model.read_slot(ring[1])
        acc = pattern(0)
        for q in range(1, world):
            acc = (acc + pattern(q)).astype(np.float32)
        rt, _, _ = O.rmsprop_update_f32(O.Hyper(), th, g0, acc)
        out["theta_bitwise"] = bool(np.array_equal(th1, rt))
        # the rms state is sharded: this rank owns shard `rank` of g
        per = -(-P // world)
        per = (per + 3) & ~3  # the kernel's shard: multiples of 4 floats (dp_fused.cuh)
        lo, hi = min(per * rank, P), min(per * rank + per, P)
        _, rg, _ = O.rmsprop_update_f32(O.Hyper(), th, g0, acc)
        out["g_shard_bitwise"] = bool(np.array_equal(g1[lo:hi], rg[lo:hi]))
    fused.close()
    dist.destroy_process_group()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
