"""Generate the committed golden vectors under tests/golden/ (run here, where
/root/reference exists; the GPU box only reads the .npz files).

  ref_mlp_*.npz   outputs of the reference's OWN nnet.cpp/returns.cpp
                  (oracle/_ref/libqac_ref.so, built from /root/reference by
                  oracle/Makefile) on the reference test shapes
                  (test_nnet.cpp:99-173) -- these pin the oracle.
  ref_returns.npz the reference's compute_returns on random segments
                  (test_returns.cpp:61-76 style).
  conv_small.npz  the oracle's conv restatement on a small strided conv net
                  (conv parity is unpinned by reference tests; this fixture
                  freezes the oracle that tests/test_oracle.py pins by the
                  bridge, finite differences and torch float64).
  dnn_a.npz       DNN A forward/loss summary on synthetic 84x84x4 frames.

Usage: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

MLP_CASES = [  # (name, input_dim, hidden, n_actions, model_seed, batch, batch_seed)
    ("ref_mlp_doc", 4, [8], 3, 202, 5, 101),       # test_nnet.cpp:158-160
    ("ref_mlp_nohidden", 3, [], 2, 404, 4, 303),   # :161-164
    ("ref_mlp_two", 5, [6, 4], 3, 606, 6, 505),    # :165-168
    ("ref_mlp_fc_tail", 2592, [256], 6, 7, 5, 9),  # DNN A's FC tail shape
]

SMALL_CONV = dict(in_hwc=(12, 12, 2), convs=[(4, 4, 2), (6, 3, 1)], hidden=[16], n_actions=3)


def ref_case(indim, hidden, A, mseed, B, bseed, hyper):
    r = O.ref()
    hid = np.array(hidden, np.int32)
    P = r.ref_param_count(indim, hid, len(hidden), A)
    th = np.zeros(P)
    r.ref_init_model(indim, hid, len(hidden), A, mseed, th)
    u = np.zeros(B * (indim + 2))
    r.ref_uniforms(bseed, u, u.size)
    st = (u[: B * indim] * 2.0 - 1.0).reshape(B, indim)
    acts = (u[B * indim: B * indim + B] * A).astype(np.int32)
    rets = u[B * indim + B:] * 4.0 - 2.0
    pi = np.zeros((B, A))
    v = np.zeros(B)
    assert r.ref_forward(indim, hid, len(hidden), A, th, P, st, B, pi, v) == 0
    d = np.zeros(P)
    sc = np.zeros(3)
    assert r.ref_loss_and_gradients(indim, hid, len(hidden), A, hyper, th, P, st, acts, rets, B, d, sc) == 0
    g0 = np.abs(d) * 0.5
    th2, g2 = np.zeros(P), np.zeros(P)
    ver = O.C.c_uint64(0)
    assert r.ref_rmsprop_update(hyper, th, g0, d, P, th2, g2, 3, O.C.byref(ver)) == 1
    return dict(input_dim=indim, hidden=np.array(hidden, np.int32), n_actions=A, model_seed=mseed,
                theta=th, states=st, actions=acts, returns=rets, pi=pi, v=v, dtheta=d, scalars=sc,
                g_in=g0, theta_out=th2, g_out=g2, version_out=ver.value)


def main():
    assert O.ref_available(), "build oracle/_ref first: make -C oracle"
    hyper = O.Hyper()
    for name, indim, hidden, A, ms, B, bs in MLP_CASES:
        case = ref_case(indim, hidden, A, ms, B, bs, hyper)
        if case["theta"].size > 100000:
            # large shape: keep theta reproducible from model_seed (init is
            # pinned bitwise on the small cases) and store fixed samples only
            idx = np.unique(np.linspace(0, case["theta"].size - 1, 3000).astype(np.int64))
            for k in ("theta", "dtheta", "g_in", "theta_out", "g_out"):
                case[k + "_sample"] = case.pop(k)[idx]
            case["idx"] = idx
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **case)

    # returns: 200 random segments through the reference
    r = O.ref()
    u = np.zeros(200 * 30)
    r.ref_uniforms(42, u, u.size)
    rows = []
    k = 0
    for _ in range(200):
        n = 1 + int(u[k] * 20); k += 1
        rew = u[k:k + n] * 20.0 - 10.0; k += n
        term = int(u[k] < 0.5); boot = u[k + 1] * 10.0 - 5.0; gamma = 0.5 + u[k + 2] * 0.5; k += 3
        out = np.zeros(n)
        assert r.ref_compute_returns(rew, n, term, boot, gamma, out) == 0
        rows.append((rew, term, boot, gamma, out))
    off = np.cumsum([0] + [len(x[0]) for x in rows]).astype(np.int32)
    np.savez_compressed(os.path.join(OUT, "ref_returns.npz"),
                        rewards=np.concatenate([x[0] for x in rows]), offsets=off,
                        terminal=np.array([x[1] for x in rows], np.uint8),
                        bootstrap=np.array([x[2] for x in rows]), gamma=np.array([x[3] for x in rows]),
                        returns=np.concatenate([x[4] for x in rows]))

    # sampler: reference sample_index draws over a fixed policy
    probs = np.array([0.1, 0.25, 0.05, 0.3, 0.2, 0.1])
    draws = np.zeros(5000, np.int32)
    r.ref_sample_many(probs, 6, 1234, 5000, draws)
    uu = np.zeros(5000)
    r.ref_uniforms(1234, uu, 5000)
    np.savez_compressed(os.path.join(OUT, "ref_sampler.npz"), probs=probs, seed=1234, u=uu, actions=draws)

    # small strided conv net through the oracle (fp64)
    sc = SMALL_CONV
    spec = O.make_spec(sc["in_hwc"], sc["convs"], sc["hidden"], sc["n_actions"])
    th = O.init_model(spec, 31)
    B = 7
    frames = O.synthetic_frames(5, B, sc["in_hwc"])
    st = O.frames_to_states(frames)
    acts, rets = O.synthetic_batch(5, B, sc["n_actions"])
    pi, v = O.forward(spec, th, st)
    d, s3 = O.loss_and_gradients(spec, hyper, th, st, acts, rets)
    np.savez_compressed(os.path.join(OUT, "conv_small.npz"), frames=frames, actions=acts, returns=rets,
                        model_seed=31, theta=th, pi=pi, v=v, dtheta=d, scalars=s3)

    # DNN A on synthetic frames: pi, v, scalars and a fixed sample of dtheta
    spec = O.dnn_a()
    th = O.init_model(spec, O.derive_seed(1, [O.SEED_MODEL_INIT]))
    th32 = th.astype(np.float32).astype(np.float64)  # the device computes on fp32 weights
    B = 4
    frames = O.synthetic_frames(1, B)
    st = O.frames_to_states(frames)
    acts, rets = O.synthetic_batch(1, B, 6)
    pi, v = O.forward(spec, th32, st)
    d, s3 = O.loss_and_gradients(spec, hyper, th32, st, acts, rets)
    idx = np.unique(np.linspace(0, d.size - 1, 4000).astype(np.int64))
    np.savez_compressed(os.path.join(OUT, "dnn_a.npz"), frames=frames, actions=acts, returns=rets,
                        pi=pi, v=v, scalars=s3, idx=idx, dtheta_sample=d[idx],
                        dtheta_norm=np.linalg.norm(d), dtheta_sum=d.sum())
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
