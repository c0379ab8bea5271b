"""The C-ABI library loads, exports every symbol include/ga3c.h declares, and
its host-only entry points agree with the reference.  CPU only: no compute
call is made without a GPU (the compute path has no CPU fallback and must
fail loudly instead)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ga3c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ga3c_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1611_06256_b200 import _abi
    names = header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(_abi.lib, n), f"{n} declared in include/ga3c.h but not exported"
    assert set(names) == set(_abi.EXPORTED), "ctypes signature table out of sync with the header"


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1611_06256_b200", "libga3c_b200.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _spec_c(spec):
    from paper_1611_06256_b200 import _abi
    s = _abi.NetSpec()
    C.memmove(C.byref(s), C.byref(spec), C.sizeof(s))
    return s


@pytest.mark.parametrize("spec", [O.dnn_a(), O.dnn_large(1), O.dnn_large(4), O.make_spec(4, [], [8], 3),
                                  O.make_spec((12, 12, 2), [(4, 4, 2), (6, 3, 1)], [16], 3)])
def test_param_count_and_init_match_oracle(spec):
    from paper_1611_06256_b200 import _abi
    s = _spec_c(spec)
    P = _abi.lib.ga3c_param_count(C.byref(s))
    assert P == O.param_count(spec)
    t64 = np.zeros(P)
    t32 = np.zeros(P, np.float32)
    assert _abi.lib.ga3c_init_params(C.byref(s), 1234, t64.ctypes.data, t32.ctypes.data) == 0
    ref = O.init_model(spec, 1234)
    assert np.array_equal(t64, ref)
    assert np.array_equal(t32, ref.astype(np.float32))


def test_validation_matches_reference_rules():
    from paper_1611_06256_b200 import _abi, qac
    for bad in (qac.NetworkSpec(0, [], 2), qac.NetworkSpec(2, [], 1), qac.NetworkSpec(2, [0], 2)):
        assert _abi.lib.ga3c_validate_spec(bad.to_c()) == _abi.INVALID_ARGUMENT
        with pytest.raises(ValueError):
            qac.param_count(bad)
    h = qac.Hyperparams()
    assert _abi.lib.ga3c_validate_hyper(h.to_c()) == 0
    for kw in (dict(gamma=0.0), dict(alpha=1.0), dict(eps_log=0.0), dict(eta=0.0)):
        assert _abi.lib.ga3c_validate_hyper(qac.Hyperparams(**kw).to_c()) == _abi.INVALID_ARGUMENT
    d = _abi.default_hyper()
    assert (d.gamma, d.t_max, d.beta, d.eta, d.alpha) == (0.99, 5, 0.01, 3e-4, 0.99)


def test_qac_api_surface_matches_reference_names():
    from paper_1611_06256_b200 import qac
    for name in ("NetworkSpec", "Hyperparams", "param_count", "init_model", "init_rms", "forward",
                 "policy_entropy", "loss_and_gradients", "rmsprop_update", "compute_returns"):
        assert hasattr(qac, name)
    assert qac.param_count(qac.NetworkSpec(4, [8], 3)) == 76
    m = qac.init_model(qac.NetworkSpec(4, [8], 3), 7)
    assert m.theta.dtype == np.float32 and m.version == 0


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1611_06256_b200 import _abi
    with pytest.raises(_abi.GA3CError):
        _abi.Model(O_spec_to_abi(), _abi.default_hyper())


def O_spec_to_abi():
    return _spec_c(O.make_spec(4, [], [8], 3))


def _resource_usage():
    """(demangled kernel name, registers) for every kernel in the library."""
    import subprocess
    so = os.path.join(ROOT, "paper_1611_06256_b200", "libga3c_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--dump-resource-usage", so], capture_output=True,
                         text=True).stdout
    mangled = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+)", out)
    names = subprocess.run(["c++filt"], input="\n".join(m for m, _ in mangled), capture_output=True,
                           text=True).stdout.splitlines()
    return [(n, int(r)) for n, (_, r) in zip(names, mangled)]


def test_two_cta_kernels_fit_two_per_sm():
    """Ring caps 1 and 2 plan two 288-thread warp-specialised CTAs per SM
    (engine.cu ring_cap).  Registers are allocated per SM sub-partition: 18
    warps put 5 on one sub-partition, so 16K / (5 * 32) -> at most 96 per
    thread.  Above that the hardware runs one CTA per SM and the planned
    overlap silently disappears (large s1 conv2 dgrad: 71 -> 112 us)."""
    rows = _resource_usage()
    checked = 0
    for name, reg in rows:
        m = re.match(r"void ga3c::(dg::tc_dgrad_kernel|ws::tc_mn_ws_kernel|ws::tc_kk_ws_kernel)<(.*)>\(", name)
        if not m:
            continue
        args = [a.strip() for a in m.group(2).split(",")]
        if m.group(1).endswith("tc_dgrad_kernel"):
            bn, cap = int(args[0]), int(args[1])
        elif m.group(1).endswith("tc_mn_ws_kernel"):
            bn, cap = int(args[1]), int(args[2])
        else:
            bn, cap = int(args[2]), int(args[4])
        if cap in (1, 2) and bn <= 64:
            checked += 1
            assert reg <= 96, f"{name}: {reg} registers -> one CTA per SM at ring cap {cap}"
    assert checked >= 10


def test_new_entry_points_reject_bad_arguments_without_a_device():
    """The round-2 entry points (trainer pool, asynchronous prediction,
    pinned host memory, engine options) check their arguments
    before touching a device: null handles and bad sizes are
    GA3C_INVALID_ARGUMENT, and no call falls back to the CPU."""
    from paper_1611_06256_b200 import _abi
    L = _abi.lib
    st = C.c_int(0)
    assert not L.ga3c_trainer_pool_create(None, None, 4, 64, 0, 16, C.byref(st))
    assert st.value == _abi.INVALID_ARGUMENT
    assert L.ga3c_trainer_pool_submit(None, None, None, 0, None, None, None, 0, None, None, 0.99) == \
        _abi.INVALID_ARGUMENT
    assert L.ga3c_trainer_pool_submit_many(None, 1, None, None, None, None, None, None, None, None, None,
                                           0.99) == _abi.INVALID_ARGUMENT
    assert L.ga3c_trainer_pool_wait(None, None, None) == _abi.INVALID_ARGUMENT
    assert L.ga3c_trainer_pool_error(None) == b""
    L.ga3c_trainer_pool_destroy(None)
    assert L.ga3c_predict_frames64_async(None, -1, None, None, None, None, 0, None) == _abi.INVALID_ARGUMENT
    assert L.ga3c_predict_collect64(None, None, None, None) == _abi.INVALID_ARGUMENT
    assert L.ga3c_ctx_set_priority(None, 1) == _abi.INVALID_ARGUMENT
    L.ga3c_host_free(None)
    opts = _abi.PipelineOpts()
    L.ga3c_default_pipeline_opts(C.byref(opts))
    assert opts.device_frames == 0 and opts.trainer_sms == -1 and opts.predictor_sms == -1
