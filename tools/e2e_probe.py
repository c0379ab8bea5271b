"""Latency of the host-buffer calls the e2e leg makes (DNN A, 1 GPU):
predict_frames (128 agents), train_frames (40 samples), apply_rmsprop,
each timed over many calls from one thread, and 16 train+apply from 4
threads as the e2e trainers do."""
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1611_06256_b200 import _abi  # noqa: E402


def main():
    import torch
    if os.environ.get("SWITCH"):
        sys.setswitchinterval(float(os.environ["SWITCH"]))
    convs, hidden = bench.NETS["dnn_a"]
    spec = _abi.NetSpec()
    spec.in_h, spec.in_w, spec.in_c = bench.FRAME
    spec.n_conv = len(convs)
    for i, (co, k, s) in enumerate(convs):
        spec.conv_out[i], spec.conv_k[i], spec.conv_stride[i] = co, k, s
    spec.n_hidden = 1
    spec.hidden[0] = 256
    spec.n_actions = 6
    hyper = _abi.default_hyper()
    model = _abi.Model(spec, hyper, 0)
    th = np.zeros(model.P, np.float32)
    _abi.check(_abi.lib.ga3c_init_params(spec, 1, None, th.ctypes.data))
    model.load(th)
    NA, T, TB = 128, 5, 40
    ctx = _abi.Context(model, NA)
    store = _abi.Frames(model, NA, 3 * T + 2)
    rng = np.random.default_rng(0)
    newf = torch.from_numpy(rng.integers(0, 256, (NA, 84 * 84), dtype=np.uint8)).pin_memory().numpy()
    agents = np.arange(NA, dtype=np.int32)
    slots = np.zeros((NA, T), np.int32)
    for t in range(T):
        _, _, sl, _ = _abi.predict_frames(ctx, store, newf, agents, None)
        slots[:, t] = sl

    def timeit(fn, n=200):
        for _ in range(10):
            fn()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        return 1e6 * (time.perf_counter() - t0) / n

    print(f"predict_frames(128): {timeit(lambda: _abi.predict_frames(ctx, store, newf, agents, None)):.1f} us")
    per = TB // T
    ag = np.repeat(agents[:per], T)
    sl = slots[:per].reshape(-1)
    acts = rng.integers(0, 6, TB).astype(np.int32)
    rew = rng.random(TB)
    seg = np.arange(0, TB + 1, T, dtype=np.int32)
    term = np.zeros(per, np.uint8)
    boot = np.zeros(per)
    tr = lambda c: _abi.train_frames(c, store, ag, sl, acts, rew, seg, term, boot, 0.99)
    print(f"train_frames(40): {timeit(lambda: tr(ctx)):.1f} us")
    print(f"apply_rmsprop: {timeit(lambda: ctx.apply_rmsprop()):.1f} us")
    print(f"train+apply: {timeit(lambda: (tr(ctx), ctx.apply_rmsprop())):.1f} us")
    for nt in (1, 2, 4, 8):
        cs = [_abi.Context(model, NA) for _ in range(nt)]
        n_upd = 160

        def worker(j):
            for _ in range(j, n_upd, nt):
                tr(cs[j])
                cs[j].apply_rmsprop()
        ths = [threading.Thread(target=worker, args=(j,)) for j in range(nt)]
        t0 = time.perf_counter()
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
        dt = time.perf_counter() - t0
        print(f"{nt} trainer threads: {1e6 * dt / n_upd:.1f} us per update (16 updates = {16e3 * dt / n_upd:.3f} ms)")
        for c in cs:
            c.close()
    # the native trainer pool (ga3c_trainer_pool_submit_many): 160 updates
    for nt in (1, 2, 4, 6, 8):
        for sms in (111, 0):
            pool = _abi.TrainerPool(model, store, nt, NA, sms, queue_cap=64)
            n_upd = 160
            b_off = np.arange(0, TB * n_upd + 1, TB, dtype=np.int32)
            s_base = np.arange(0, per * n_upd + 1, per, dtype=np.int32)
            pool.submit_many(b_off[:17], s_base[:17], np.tile(ag, 16), np.tile(sl, 16), np.tile(acts, 16),
                             np.tile(rew, 16), np.tile(seg, 16), np.tile(term, 16), np.tile(boot, 16), 0.99)
            pool.wait()
            t0 = time.perf_counter()
            pool.submit_many(b_off, s_base, np.tile(ag, n_upd), np.tile(sl, n_upd), np.tile(acts, n_upd),
                             np.tile(rew, n_upd), np.tile(seg, n_upd), np.tile(term, n_upd), np.tile(boot, n_upd),
                             0.99)
            pool.wait()
            dt = time.perf_counter() - t0
            print(f"native pool, {nt} threads, sms {sms}: {1e6 * dt / n_upd:.1f} us per update "
                  f"(16 updates = {16e3 * dt / n_upd:.3f} ms)", flush=True)
            pool.close()
    # raw C call overhead: an empty predict (n = 0)
    print(f"predict_frames(0): {timeit(lambda: _abi.predict_frames(ctx, store, newf[:0], agents[:0], None)):.1f} us")


if __name__ == "__main__":
    main()
