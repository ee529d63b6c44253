"""Parity of every plan bench.py times, at the timed size.

Each test builds its plan with ``bench.make_device_plan`` — the exact call the
benchmark times — asserts the device factorisation it executes, runs it on
device-resident buffers (the timed path) and compares the result with the
reference's own ``fft_tiled`` (oracle/_ref: the reference headers compiled
unmodified, tiled_fft.hpp:321-407) on the same fp32 input, within the north-star
tolerance rel L2 <= 1e-5 * log2 N (the measured errors are ~1e-7, so each test
also asserts < 5e-7). No environment switch is set: these are the default plans.

* 2^26 single transform   (BASELINE configs[2]) vs fft_tiled(x, make_plan(2^26, 1024))
* 8192 x 8192 image       (configs[3]) vs the reference rows-then-columns
* 2^30 single transform   (configs[4], one GPU) vs fp32 fft_tiled + 16 exact fp64 bins
* 2^30 over 2/4/8 virtual ranks (configs[4], the distributed four-step kernels on one
  B200) vs the same reference output
"""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_lib import rel_l2  # noqa: E402

THREADS = os.cpu_count() or 8


def tol(n):
    return 1e-5 * math.log2(n)


@pytest.fixture(autouse=True)
def _default_plans(monkeypatch):
    for k in list(os.environ):
        if k.startswith("TILEFFT_"):
            monkeypatch.delenv(k)


def _run_device(plan, x: np.ndarray) -> np.ndarray:
    import torch
    from paper_1707_07263_b200 import _capi
    xd = torch.from_numpy(x.view(np.float32)).cuda()
    yd = torch.empty_like(xd)
    plan.exec_device(xd.data_ptr(), yd.data_ptr(), _capi.FORWARD, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    y = yd.cpu().numpy().view(np.complex64).reshape(x.shape)
    del xd, yd
    torch.cuda.empty_cache()
    return y


def test_1d_2e26_bench_plan_vs_reference(reference):
    import bench
    n = 1 << 26
    plan = bench.make_device_plan("1d_2e26")
    info = plan.info()
    assert info["factors"] == bench.DEVICE_FACTORS["1d_2e26"], info["factors"]
    x = reference.random_bench_signal(n, 1).astype(np.complex64)
    got = _run_device(plan, x)
    want = reference.fft_tiled(x, 1024, threads=THREADS)  # make_plan(2^26, 1024) = [512, 512, 256]
    err = rel_l2(got, want)
    assert err <= tol(n), err
    assert err < 5e-7, err


def test_2d_8192_bench_plan_vs_reference_rows_then_columns(reference, oracle):
    import bench
    n = 8192
    plan = bench.make_device_plan("2d_8192")
    info = plan.info()
    assert info["factors"] == bench.DEVICE_FACTORS["2d_8192"], info["factors"]
    img = oracle.splitmix_signal(n * n, 3).reshape(n, n)
    got = _run_device(plan, img)
    want = reference.fft2(img, 1024, threads=THREADS)
    err = rel_l2(got, want)
    assert err <= tol(n * n), err
    assert err < 5e-7, err


# ---- 2^30: one reference run shared by the single-GPU and the distributed tests -------------------
@pytest.fixture(scope="module")
def ref_2e30(reference, oracle):
    n = 1 << 30
    x = oracle.splitmix_signal(n, 7)  # counter-based input (SURVEY §8d, 2^30 row)
    want = reference.fft_tiled(x, 1024, threads=THREADS)  # make_plan(2^30, 1024) = [1024]^3
    bins = np.array([0, 1, 2, 3, 1023, 1024, 65537, 1 << 20, (1 << 29) - 1, 1 << 29, (1 << 29) + 1,
                     123456789, 987654321, (1 << 30) - 1024, (1 << 30) - 2, (1 << 30) - 1], dtype=np.uint64)
    exact = oracle.dft_bins(x, bins, threads=THREADS)
    rms = math.sqrt(n * float(np.mean(np.abs(x[: 1 << 22].astype(np.complex128)) ** 2)))  # |X| scale
    # the reference itself against the exact bins (pins the oracle at this size)
    assert np.max(np.abs(want[bins.astype(np.int64)] - exact)) / rms < 1e-5 * 30
    return x, want, bins, exact, rms


def _check_2e30(got, ref):
    x, want, bins, exact, rms = ref
    n = x.shape[-1]
    err = rel_l2(got, want)
    assert err <= tol(n), err
    assert err < 5e-7, err
    binerr = float(np.max(np.abs(got[bins.astype(np.int64)] - exact))) / rms
    assert binerr <= tol(n), binerr


def test_1d_2e30_bench_plan_vs_reference(ref_2e30):
    import bench
    plan = bench.make_device_plan("1d_2e30")
    info = plan.info()
    assert info["factors"] == bench.DEVICE_FACTORS["1d_2e30"], info["factors"]
    got = _run_device(plan, ref_2e30[0])
    del plan
    _check_2e30(got, ref_2e30)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_1d_2e30_distributed_virtual_ranks_vs_reference(ref_2e30, world):
    """The distributed four-step kernels (pass 1 scattering into the owners'
    row slabs = the all-to-all, then the local row passes) for G ranks, run as
    G plans on one B200 writing each other's slabs."""
    import torch
    from paper_1707_07263_b200 import _capi
    from paper_1707_07263_b200.distributed import assemble_output, four_step_layout
    x = ref_2e30[0]
    n = x.shape[-1]
    n1, n2, c, r = four_step_layout(n, world)
    plans = [_capi.DistPlan.create_dist(n, world, g, 8, 0) for g in range(world)]
    rows = [torch.zeros((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)]
    for g, p in enumerate(plans):
        p.set_peers([t.data_ptr() for t in rows], n2, g * c)
    xv = x.reshape(n1, n2)
    for g, p in enumerate(plans):
        slab = torch.from_numpy(np.ascontiguousarray(xv[:, g * c:(g + 1) * c])).cuda()
        p.pass1(slab.data_ptr())
        torch.cuda.synchronize()
        del slab
    outs = []
    for g, p in enumerate(plans):
        o = torch.empty_like(rows[g])
        p.pass2(rows[g].data_ptr(), o.data_ptr())
        torch.cuda.synchronize()
        outs.append(o.cpu().numpy())
        del o
    del rows, plans
    torch.cuda.empty_cache()
    got = assemble_output(outs, n)
    del outs
    _check_2e30(got, ref_2e30)


def test_1d_2e26_bench_plan_inverse_and_host_path(reference):
    """The 2^26 plan's inverse (ifft_tiled: conjugate trick + 1/n, tiled_fft.hpp:410-423) vs the reference's
    own ifft on the same input, and the host-buffer entry point (the e2e leg) bitwise equal to the device path."""
    import torch
    import bench
    from paper_1707_07263_b200 import _capi
    n = 1 << 26
    plan = bench.make_device_plan("1d_2e26")
    x = reference.random_bench_signal(n, 4).astype(np.complex64)
    xd = torch.from_numpy(x.view(np.float32)).cuda()
    yd = torch.empty_like(xd)
    plan.exec_device(xd.data_ptr(), yd.data_ptr(), _capi.INVERSE, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = yd.cpu().numpy().view(np.complex64)
    want = reference.fft_tiled(x, 1024, threads=THREADS, inverse=True)
    err = rel_l2(got, want)
    assert err <= tol(n) and err < 5e-7, err
    hout = np.empty_like(x)
    plan.exec_host(x.ctypes.data, hout.ctypes.data, _capi.INVERSE)
    assert np.array_equal(hout.view(np.uint32), got.view(np.uint32))
    del xd, yd
    torch.cuda.empty_cache()


def test_2d_8192_bench_plan_inverse_roundtrip(oracle):
    """ifft2(fft2(x)) == x on the timed 8192^2 plan (both directions through the two-level column pass)."""
    import torch
    import bench
    from paper_1707_07263_b200 import _capi
    n = 8192
    plan = bench.make_device_plan("2d_8192")
    x = oracle.splitmix_signal(n * n, 5)
    xd = torch.from_numpy(x.view(np.float32)).cuda()
    yd = torch.empty_like(xd)
    st = torch.cuda.current_stream().cuda_stream
    plan.exec_device(xd.data_ptr(), yd.data_ptr(), _capi.FORWARD, st)
    plan.exec_device(yd.data_ptr(), yd.data_ptr(), _capi.INVERSE, st)
    torch.cuda.synchronize()
    back = yd.cpu().numpy().view(np.complex64)
    err = rel_l2(back, x)
    assert err <= tol(n * n) and err < 1e-6, err
    del xd, yd
    torch.cuda.empty_cache()
