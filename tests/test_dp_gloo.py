"""Data-parallel semantics on CPU with the gloo backend, world_size 2.

Each rank computes the oracle's summed gradient on its shard of a merged
training batch; an all-reduce(sum) must reproduce the whole-batch gradient
(the reference sums, nnet.hpp:88-94), the clip is applied after the
reduction, and identical RMSProp steps keep the replicas bit-identical.
This is the host-side contract paper_1611_06256_b200/dp.py implements on
the GPU box with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import pyoracle as O

SPEC = O.make_spec((12, 12, 2), [(4, 4, 2)], [8], 4)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, clip):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    from paper_1611_06256_b200.dp import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hp = O.Hyper(grad_clip_norm=clip)
    th = O.init_model(SPEC, 5)
    B = 9
    fr = O.synthetic_frames(11, B, (12, 12, 2))
    st = O.frames_to_states(fr)
    acts, rets = O.synthetic_batch(11, B, 4)
    lo, hi = shard(B, rank, world)
    hp_noclip = O.Hyper()
    d, _ = O.loss_and_gradients(SPEC, hp_noclip, th, st[lo:hi], acts[lo:hi], rets[lo:hi])
    t = torch.from_numpy(d.copy())
    dist.all_reduce(t)  # ncclSum on the GPU box
    g = t.numpy()
    if clip > 0:  # global-norm clip on the reduced gradient (nnet.cpp:281-289)
        n = np.sqrt(np.sum(g * g))
        if n > clip:
            g = g * (clip / n)
    th2, g2, ok = O.rmsprop_update(hp, th, np.zeros_like(th), g)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.stack([g, th2]))
    dist.destroy_process_group()


@pytest.mark.parametrize("clip", [0.0, 0.05])
def test_dp_allreduce_reproduces_single_device_step(tmp_path, clip):
    world = 2
    mp.start_processes(_worker, args=(world, _port(), str(tmp_path), clip), nprocs=world, start_method="spawn")
    r0 = np.load(tmp_path / "r0.npy")
    r1 = np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1)  # replicas identical after the step
    th = O.init_model(SPEC, 5)
    B = 9
    fr = O.synthetic_frames(11, B, (12, 12, 2))
    acts, rets = O.synthetic_batch(11, B, 4)
    d, _ = O.loss_and_gradients(SPEC, O.Hyper(grad_clip_norm=clip), th, O.frames_to_states(fr), acts, rets)
    assert np.allclose(r0[0], d, rtol=1e-12, atol=1e-14)
    th_ref, _, _ = O.rmsprop_update(O.Hyper(grad_clip_norm=clip), th, np.zeros_like(th), d)
    assert np.allclose(r0[1], th_ref, rtol=0, atol=1e-12)


def test_shards_and_agent_sharding():
    from paper_1611_06256_b200.dp import agents_of, shard
    for n in (1, 5, 40, 41):
        for world in (1, 2, 4, 8):
            parts = [shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
    assert sorted(sum((agents_of(r, 4, 10) for r in range(4)), [])) == list(range(10))


def test_peer_lists_keep_own_pointers_and_open_peers():
    """FusedUpdate's IPC wiring: index = rank; this rank's own buffers as they
    are, every peer's through the opener (CUDA IPC on the GPU box)."""
    from paper_1611_06256_b200 import dp

    world, rank = 3, 1
    gathered = [{"grad": [f"g{q}a", f"g{q}b"], "sig": [f"s{q}"]} for q in range(world)]
    local = {"grad": [100, 101], "sig": [200]}
    opened = []
    lists = dp.peer_lists(local, gathered, rank, lambda h: opened.append(h) or f"open({h})")
    assert lists["grad"][0] == ["open(g0a)", 100, "open(g2a)"]
    assert lists["grad"][1] == ["open(g0b)", 101, "open(g2b)"]
    assert lists["sig"][0] == ["open(s0)", 200, "open(s2)"]
    assert sorted(opened) == sorted(["g0a", "g2a", "g0b", "g2b", "s0", "s2"])
