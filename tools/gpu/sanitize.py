"""Small transforms through the round-2 kernels, for compute-sanitizer (memcheck / racecheck /
synccheck): the two-level pass k_two_tma (plain columns with B-side roots, both output layouts of the
four-step 1D plan, inverse), the persistent final pass k_final_p, the prefetching long-row kernel, the
three-half-slot comb kernel k_comb_h3 and the transposed pass-0 -> pass-1 hand-over of 3-pass plans.
(The distributed barrier kernel waits for kernels on other streams, which the sanitizer serialises.)"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_1707_07263_b200 import _capi
from oracle_lib import Oracle, rel_l2

orc = Oracle()

def run2d(ny, nx, sign=_capi.FORWARD):
    img = orc.random_bench_signal(ny * nx, 3).astype(np.complex64).reshape(ny, nx)
    dp = _capi.DevicePlan.create_2d(ny, nx, 1, 8, 0)
    out = np.empty_like(img)
    dp.exec_host(img.ctypes.data, out.ctypes.data, sign)
    if sign == _capi.FORWARD:
        e = rel_l2(out, orc.fft2(img))
        print(f"2d {ny}x{nx} rel_l2 {e:.2e}", flush=True)
        assert e < 1e-5 * np.log2(ny * nx)
    dp.close()

def run1d(n, env):
    os.environ.update(env)
    x = orc.random_bench_signal(n, 5).astype(np.complex64)
    dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
    out = np.empty_like(x)
    dp.exec_host(x.ctypes.data, out.ctypes.data, _capi.FORWARD)
    e = rel_l2(out, orc.fft_tiled(x))
    print(f"1d {n} {env} factors {dp.info()['factors']} rel_l2 {e:.2e}", flush=True)
    assert e < 1e-5 * np.log2(n)
    dp.close()
    for k in env: os.environ.pop(k)

def run1db(n, b):
    x = orc.random_bench_signal(n * b, 6).astype(np.complex64).reshape(b, n)
    dp = _capi.DevicePlan.create(n, b, None, 8, _capi.MODE_FAST, None, 0)
    out = np.empty_like(x)
    dp.exec_host(x.ctypes.data, out.ctypes.data, _capi.FORWARD)
    e = rel_l2(out, orc.fft_tiled(x))
    print(f"1d {n} x {b} factors {dp.info()['factors']} rel_l2 {e:.2e}", flush=True)
    assert e < 1e-5 * np.log2(n)
    dp.close()

run1db(1 << 19, 16)   # [1024, 512]: k_comb_h3<1024>
run1d(1 << 25, {})    # [512, 256, 256]: k_comb_h3<512> with the transposed store, in_t pass 1
run2d(2048, 32)
run2d(2048, 32, _capi.INVERSE)
run2d(256, 2048)
run1d(1 << 22, {"TILEFFT_TWO_1D": "1"})
run1d(1 << 22, {})
run1d(8192, {})
print("sanitize workload ok")
