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
