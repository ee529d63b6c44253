"""The C-ABI library: loads, exports every symbol include/tilefft_b200.h
declares, and refuses to run without a GPU (no CPU fallback). CPU only — no
compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tilefft_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"TILEFFT_API\s+[\w\s\*]+?\b(tilefft_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1707_07263_b200 import _capi
    return _capi.load()


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for s in ("tilefft_plan_create", "tilefft_exec_c2c", "tilefft_exec_c2c_host", "tilefft_plan_destroy",
              "tilefft_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_1707_07263_b200 import _capi
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert sorted(_capi.EXPORTS) == header_symbols()
    assert lib.tilefft_version().decode().startswith("tilefft_b200")


def test_library_is_sm100a(lib):
    import subprocess
    so = os.path.join(ROOT, "paper_1707_07263_b200", "libtilefft_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1707_07263_b200 import _capi
    h = ctypes.c_void_p()
    rc = lib.tilefft_plan_create(ctypes.byref(h), 1024, 1, None, 0, 8, 0, None, 0, 0)
    assert rc == _capi.ENODEV
    assert "no CUDA device" in lib.tilefft_last_error().decode()
    import numpy as np
    import paper_1707_07263_b200 as tf
    with pytest.raises(_capi.TilefftError):
        tf.fft_tiled(np.zeros(1024, np.complex64), tf.make_plan(1024))


def test_argument_errors_are_einval(lib):
    from paper_1707_07263_b200 import _capi
    h = ctypes.c_void_p()
    assert lib.tilefft_plan_create(ctypes.byref(h), 48, 1, None, 0, 8, 0, None, 0, 0) == _capi.EINVAL
    assert "n must be a power of two" in lib.tilefft_last_error().decode()
    f = (ctypes.c_uint64 * 2)(4, 4)
    assert lib.tilefft_plan_create(ctypes.byref(h), 32, 1, f, 2, 8, 1, None, 0, 0) == _capi.EINVAL
    assert "does not match the plan" in lib.tilefft_last_error().decode()
    assert lib.tilefft_plan_create(ctypes.byref(h), 32, 1, None, 0, 8, 1, None, 0, 0) == _capi.EINVAL
    assert "empty plan" in lib.tilefft_last_error().decode()
    assert lib.tilefft_exec_c2c(None, None, None, -1, None) == _capi.EINVAL


def test_round2_entry_points_reject_bad_arguments(lib):
    """Null-plan / null-buffer / bad-argument paths of the round-2 entry points return EINVAL with a message
    (no device work, so this runs without a GPU too)."""
    from paper_1707_07263_b200 import _capi
    ms = (ctypes.c_float * 4)()
    assert lib.tilefft_exec_c2c_timed(None, None, None, -1, None, 1, ms, 4) == _capi.EINVAL
    assert "null plan" in lib.tilefft_last_error().decode()
    assert lib.tilefft_dist_exec(None, None, None, -1, None) == _capi.EINVAL
    assert "not a distributed plan" in lib.tilefft_last_error().decode()
    assert lib.tilefft_dist_exec_pass2_blocks(None, None, None, -1, None) == _capi.EINVAL
    assert lib.tilefft_dist_set_flags(None, None, 0) == _capi.EINVAL
    p = ctypes.c_void_p()
    assert lib.tilefft_dist_flag_buffer(None, ctypes.byref(p)) == _capi.EINVAL
    assert lib.tilefft_ipc_get_handle(None, None, None) == _capi.EINVAL
    assert lib.tilefft_ipc_open_handle(None, 0, None) == _capi.EINVAL


@pytest.mark.gpu
def test_timed_exec_and_dist_guards(lib):
    """exec_c2c_timed reports one positive time per pass; a distributed plan refuses tilefft_dist_exec until its
    barrier words are set and rejects a flag list whose own entry is not its own buffer."""
    import torch
    from paper_1707_07263_b200 import _capi
    dp = _capi.DevicePlan.create(1 << 20, 1, None, 8, _capi.MODE_FAST, None, 0)
    x = torch.randn(1 << 20, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    ms = dp.exec_timed(x.data_ptr(), y.data_ptr(), reps=3)
    assert len(ms) == dp.info()["passes"] == 2 and all(v > 0 for v in ms)
    with pytest.raises(ValueError, match="reps"):
        _capi.check(lib.tilefft_exec_c2c_timed(dp._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                               -1, None, 0, (ctypes.c_float * 2)(), 2))
    d0 = _capi.DistPlan.create_dist(1 << 20, 2, 0, 8, 0)
    d1 = _capi.DistPlan.create_dist(1 << 20, 2, 1, 8, 0)
    with pytest.raises(ValueError, match="barrier flags not set"):
        d0.exec_step(x.data_ptr(), y.data_ptr())
    with pytest.raises(ValueError, match="own flag buffer"):
        d0.set_flags([d1.flag_buffer(), d0.flag_buffer()])
