"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Tiers:
  1. FAST mode: relative L2 <= 1e-5*log2(N) (fp32), 1e-12*log2(N) (fp64)
     against the reference's fft_tiled on the same input (north-star tolerance).
  2. EXACT mode: bit-identical to fft_tiled<Real> for the same plan and table.
  3. PERMUTE mode: index maps bit-exact (ramp input, butterflies off).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_lib import rel_l2  # noqa: E402


@pytest.fixture(scope="module")
def tf():
    import paper_1707_07263_b200 as tf
    return tf


def tol(n, dtype):
    return (1e-5 if dtype == np.complex64 else 1e-12) * math.log2(n)


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint8), np.ascontiguousarray(b).view(np.uint8))


# the 12 plans of test_tiled_fft.cpp:208-224 plus the BASELINE shapes (reduced where the oracle is slow)
PLANS = [(2, 1024), (4, 2), (8, 4), (16, 4), (32, 2), (64, 4), (64, 8), (256, 16), (512, 8), (1024, 4),
         (1024, 32), (1024, 1024), (4096, 64), (8192, 1024), (65536, 1024), (1 << 20, 1024), (1 << 20, 8192)]


@pytest.mark.parametrize("n,cap", PLANS)
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_exact_mode_bit_identical(tf, oracle, n, cap, dtype):
    x = oracle.random_bench_signal(n, 1).astype(dtype)
    plan = tf.make_plan(n, cap)
    table = tf.build_twiddle_table(n, dtype)
    got = tf.fft_tiled(x, plan, table, mode="exact")
    want = oracle.fft_tiled(x, cap)
    assert bits_equal(got, want), f"n={n} cap={cap} rel={rel_l2(got, want)}"


@pytest.mark.parametrize("n,cap", [(256, 16), (4096, 64), (1 << 16, 1024)])
def test_exact_mode_inverse_bit_identical(tf, oracle, n, cap):
    x = oracle.random_bench_signal(n, 2).astype(np.complex64)
    plan = tf.make_plan(n, cap)
    table = tf.build_twiddle_table(n, np.complex64)
    assert bits_equal(tf.ifft_tiled(x, plan, table, mode="exact"), oracle.fft_tiled(x, cap, inverse=True))


def test_exact_mode_larger_table_resolution(tf, oracle):
    # the table may be finer than n (tiled_fft.hpp:328-329): values are resolution independent
    n, cap, res = 4096, 64, 1 << 16
    x = oracle.random_bench_signal(n, 5).astype(np.complex64)
    got = tf.fft_tiled(x, tf.make_plan(n, cap), tf.build_twiddle_table(res, np.complex64), mode="exact")
    assert bits_equal(got, oracle.fft_tiled(x, cap, res=res))


def test_exact_mode_batched(tf, oracle):
    n, cap, b = 1024, 32, 7
    x = np.stack([oracle.random_signal(n, 100 + i) for i in range(b)]).astype(np.complex64)
    got = tf.fft_tiled(x, tf.make_plan(n, cap), tf.build_twiddle_table(n, np.complex64), mode="exact")
    assert bits_equal(got, oracle.fft_tiled(x, cap))


@pytest.mark.parametrize("n,cap", [(16, 4), (8, 4), (64, 4), (4096, 64), (1 << 20, 1024)])
def test_permute_mode_index_maps(tf, oracle, n, cap):
    ramp = np.arange(n, dtype=np.float32).astype(np.complex64)
    got = tf.fft_tiled(ramp, tf.make_plan(n, cap), None, mode="permute")
    want = oracle.permute_tiled(ramp, cap)
    assert bits_equal(got, want)
    # and the permutation is the composition of the reference's maps
    assert sorted(got.real.astype(np.int64).tolist()) == list(range(n))


FAST_SIZES = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 1 << 14, 1 << 15, 1 << 16, 1 << 17,
              1 << 18, 1 << 20]


@pytest.mark.parametrize("n", FAST_SIZES)
def test_fast_mode_fp32_within_tolerance(tf, oracle, n):
    x = oracle.random_bench_signal(n, 1).astype(np.complex64)
    got = tf.fft_tiled(x, tf.make_plan(n))
    want = oracle.fft_tiled(x)
    err = rel_l2(got, want)
    assert err <= tol(n, np.complex64), err
    assert err < 5e-7, err  # much tighter than the contract: accurate roots


@pytest.mark.parametrize("n", [2, 64, 1024, 8192, 1 << 14, 1 << 16, 1 << 20, 1 << 22])
def test_fast_mode_fp64_within_tolerance(tf, oracle, n):
    x = oracle.random_bench_signal(n, 1)
    got = tf.fft_tiled(x, tf.make_plan(n))
    err = rel_l2(got, oracle.fft_tiled(x))
    assert err <= tol(n, np.complex128), err


@pytest.mark.parametrize("n", [1024, 1 << 16, 1 << 20, 1 << 23])
def test_fast_mode_inverse(tf, oracle, n):
    x = oracle.random_bench_signal(n, 4).astype(np.complex64)
    got = tf.ifft_tiled(x, tf.make_plan(n))
    want = oracle.fft_tiled(x, inverse=True)
    assert rel_l2(got, want) <= tol(n, np.complex64)
    back = tf.ifft_tiled(tf.fft_tiled(x, tf.make_plan(n)), tf.make_plan(n))
    assert rel_l2(back, x) <= tol(n, np.complex64)


def test_fast_batched_1024_headline_shape(tf, oracle):
    """configs[1]: batched 1024 x 65536 — every row against the oracle."""
    n, b = 1024, 65536
    x = oracle.random_bench_signal(n * b, 1).astype(np.complex64).reshape(b, n)
    got = tf.fft_tiled(x, tf.make_plan(n))
    want = oracle.fft_tiled(x)
    assert rel_l2(got, want) <= tol(n, np.complex64)
    per_row = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per_row.max() < 1e-6


def test_fast_device_path_matches_host_path(tf, oracle):
    import torch
    n, b = 1 << 20, 2
    x = oracle.random_bench_signal(n * b, 9).astype(np.complex64).reshape(b, n)
    host = tf.fft_tiled(x, tf.make_plan(n))
    xd = torch.from_numpy(x).cuda()
    dev = tf.fft_tiled_device(xd, tf.make_plan(n)).cpu().numpy()
    assert bits_equal(host, dev)
    # in place
    tf.fft_tiled_device(xd, tf.make_plan(n), out=xd)
    assert bits_equal(host, xd.cpu().numpy())


def test_fast_2d_matches_rows_then_columns(tf, oracle):
    for ny, nx in [(64, 32), (1024, 1024), (2048, 512), (16, 8192)]:
        img = oracle.random_bench_signal(ny * nx, 3).astype(np.complex64).reshape(ny, nx)
        got = tf.fft2_tiled(img)
        want = oracle.fft2(img)
        assert rel_l2(got, want) <= tol(ny * nx, np.complex64), (ny, nx)


def test_fast_2d_inverse_roundtrip(tf, oracle):
    img = oracle.random_bench_signal(4096 * 256, 3).astype(np.complex64).reshape(2, 2048, 256)
    back = tf.fft2_tiled(tf.fft2_tiled(img), inverse=True)
    assert rel_l2(back, img) <= tol(2048 * 256, np.complex64)


def test_errors_match_reference(tf):
    plan = tf.make_plan(256, 16)
    x = np.zeros(128, np.complex64)
    with pytest.raises(ValueError, match="signal length does not match the plan"):
        tf.fft_tiled(x, plan)
    with pytest.raises(ValueError, match="must divide the table resolution"):
        tf.fft_tiled(np.zeros(256, np.complex64), plan, tf.build_twiddle_table(64, np.complex64))


@pytest.mark.parametrize("n", [2, 8, 1024, 1 << 16, 1 << 20])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_levelwise_gpu_bit_identical(tf, oracle, n, dtype):
    x = oracle.random_bench_signal(n, 1).astype(dtype)
    got = tf.fft_levelwise(x, tf.build_twiddle_table(n, dtype))
    assert bits_equal(got, oracle.fft_levelwise(x))


def test_levelwise_inverse_roundtrip(tf, oracle):
    n = 4096
    x = oracle.random_bench_signal(n, 2)
    t = tf.build_twiddle_table(n)
    assert rel_l2(tf.ifft_levelwise(tf.fft_levelwise(x, t), t), x) < 1e-14


def test_exchange_transpose_gpu(tf, oracle, reference):
    for n, cap in [(16, 4), (8, 4), (64, 4), (4096, 64)]:
        plan = tf.make_plan(n, cap)
        ramp = np.arange(n, dtype=np.float64).astype(np.complex128)
        for s in range(1, plan.pass_count() + 1):
            assert np.array_equal(tf.exchange_transpose(ramp, s, plan), reference.exchange_transpose(ramp, cap, s))


def test_stage_row_fft_and_interstage(tf, oracle):
    table = tf.build_twiddle_table(64)
    buf = tf.FastBuffer(2, 8, 9, 16)
    r0, r1 = oracle.random_signal(8, 21), oracle.random_signal(8, 22)
    buf.cells[0, :8], buf.cells[1, :8] = r0, r1
    tf.stage_row_fft(buf, 8, table)
    assert np.max(np.abs(buf.tile()[0] - oracle.dft(r0))) < 1e-12
    assert np.max(np.abs(buf.tile()[1] - oracle.dft(r1))) < 1e-12
    plan = tf.make_plan(4, 2)
    b = tf.make_stage_buffer(plan, 1)
    b.set_row_offset(1)
    b.cells[0, :2] = [1.0, 1.0]
    tf.apply_interstage_twiddles(b, 1, plan, tf.build_twiddle_table(16))
    assert b.tile()[0, 0] == 1.0 and b.tile()[0, 1] == -1j


@pytest.mark.parametrize("n,b", [(2048, 300), (4096, 129), (8192, 64)])
def test_fast_batched_long_rows_prefetch_kernel(tf, oracle, monkeypatch, n, b):
    """k_rows_pf (persistent long rows, next row streamed into the exchange region):
    batched through the chunked host pipeline (in place per chunk) and on device
    buffers, every row against the oracle, and bitwise equal to k_rows."""
    import torch
    x = oracle.random_bench_signal(n * b, 6).astype(np.complex64).reshape(b, n)
    want = oracle.fft_tiled(x)
    got = tf.fft_tiled(x, tf.make_plan(n))
    per_row = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per_row.max() < 1e-6
    xd = torch.from_numpy(x).cuda()
    dev = tf.fft_tiled_device(xd, tf.make_plan(n)).cpu().numpy()
    assert bits_equal(dev, got)
    # an 8-byte-aligned device buffer takes the non-persistent k_rows kernel: same bits
    buf = torch.zeros(n * b + 1, dtype=torch.complex64, device="cuda")
    buf[1:] = xd.reshape(-1)
    unal = tf.fft_tiled_device(buf[1:].view(b, n), tf.make_plan(n)).cpu().numpy()
    assert bits_equal(unal, got)


@pytest.mark.parametrize("case", ["1d_2e22", "2d_4096x512"])
def test_one_plan_two_streams_concurrently(tf, oracle, case):
    """Execs of one plan on two streams share its workspace / two-level scratch
    and counters: the plan orders them on the device, so launching both without
    any host synchronisation gives bitwise the serial results."""
    import torch
    from paper_1707_07263_b200 import _capi
    if case == "1d_2e22":
        n = 1 << 22
        dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
    else:
        n = 4096 * 512
        dp = _capi.DevicePlan.create_2d(4096, 512, 1, 8, 0)
    xs = [torch.from_numpy(oracle.random_bench_signal(n, s).astype(np.complex64)).cuda() for s in (1, 2, 3, 4)]
    serial = []
    for x in xs:
        y = torch.empty_like(x)
        dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        serial.append(y.cpu().numpy())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for rep in range(3):
        ys = [torch.empty_like(x) for x in xs]
        for i, (x, y) in enumerate(zip(xs, ys)):
            dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, streams[i % 2].cuda_stream)
        torch.cuda.synchronize()
        for y, want in zip(ys, serial):
            assert bits_equal(y.cpu().numpy(), want), rep


@pytest.mark.gpu
@pytest.mark.parametrize("n,b", [(1 << 18, 8), (1 << 22, 2), (1 << 14, 64)])
def test_fast_batched_multipass_inplace_comb(tf, oracle, n, b):
    """Batched multi-pass plans through the in-place-exchange TMA comb kernel and the persistent final pass:
    every transform against the oracle, device path == host path, and an 8-byte-aligned input (no TMA: the
    register comb kernel) within the same tolerance."""
    import torch
    x = oracle.random_bench_signal(n * b, 12).astype(np.complex64).reshape(b, n)
    want = oracle.fft_tiled(x)
    got = tf.fft_tiled(x, tf.make_plan(n))
    per = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per.max() < 5e-7, per.max()
    xd = torch.from_numpy(x).cuda()
    assert bits_equal(tf.fft_tiled_device(xd, tf.make_plan(n)).cpu().numpy(), got)
    buf = torch.zeros(n * b + 1, dtype=torch.complex64, device="cuda")
    buf[1:] = xd.reshape(-1)
    un = buf[1:].view(b, n)
    assert un.data_ptr() % 16 == 8
    tf.tilefft._plan_cache.clear()
    got_u = tf.fft_tiled_device(un, tf.make_plan(n)).cpu().numpy()
    tf.tilefft._plan_cache.clear()
    per_u = np.linalg.norm(got_u - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per_u.max() < 5e-7, per_u.max()


@pytest.mark.gpu
@pytest.mark.parametrize("n,b,dtype", [(1 << 21, 4, np.complex64), (1 << 22, 2, np.complex64),
                                       (1 << 24, 1, np.complex64), (1 << 21, 2, np.complex128)])
def test_fast_transposed_handover(tf, oracle, monkeypatch, n, b, dtype):
    """3-pass plans hand over from pass 0 to pass 1 through the transposed T[c1][k0][c2] layout
    (CombArgs::t_l2, the default): every transform against the oracle (forward, inverse), device path ==
    host path, and a misaligned input (register comb kernel for pass 0) within the same tolerance; the plan
    carries the second workspace. Then the same transforms with the in-place hand-over (TILEFFT_TSTORE=0)."""
    import torch
    for k in [k for k in __import__("os").environ if k.startswith("TILEFFT_")]:
        monkeypatch.delenv(k)
    tf.tilefft._plan_cache.clear()
    x = oracle.random_bench_signal(n * b, 21).astype(dtype).reshape(b, n)
    want = oracle.fft_tiled(x)
    plan = tf.make_plan(n)
    got = tf.fft_tiled(x, plan)
    lim = 5e-7 if dtype == np.complex64 else 1e-13
    per = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per.max() < lim, per.max()
    back = tf.ifft_tiled(got, plan)
    assert rel_l2(back, x) < (1e-6 if dtype == np.complex64 else 1e-14)
    xd = torch.from_numpy(x).cuda()
    assert bits_equal(tf.fft_tiled_device(xd, plan).cpu().numpy(), got)
    xi = xd.clone()
    tf.fft_tiled_device(xi, plan, out=xi)  # in == out: pass 0 reads the user buffer, the final pass rewrites it
    assert bits_equal(xi.cpu().numpy(), got)
    info = tf.tilefft._plan_cache and next(iter(tf.tilefft._plan_cache.values())).info()
    if info:
        assert len(info["factors"]) == 3, info
        assert info["workspace_bytes"] >= 2 * n * b * x.itemsize, info
    buf = torch.zeros(n * b + 1, dtype=xd.dtype, device="cuda")
    buf[1:] = xd.reshape(-1)
    un = buf[1:].view(b, n)
    tf.tilefft._plan_cache.clear()
    got_u = tf.fft_tiled_device(un, tf.make_plan(n)).cpu().numpy()
    tf.tilefft._plan_cache.clear()
    per_u = np.linalg.norm(got_u - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per_u.max() < lim, per_u.max()
    monkeypatch.setenv("TILEFFT_TSTORE", "0")
    got0 = tf.fft_tiled(x, tf.make_plan(n))
    tf.tilefft._plan_cache.clear()
    per0 = np.linalg.norm(got0 - want, axis=1) / np.linalg.norm(want, axis=1)
    assert per0.max() < lim, per0.max()
