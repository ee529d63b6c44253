"""The reference's cost model on the drop-in headers, host only.

include/tilefft/{exec_model,access_patterns,memsim}.hpp restate the request
primitives, request shapes and closed-form accounting of
/root/reference/proj/include/tilefft/{exec_model,access_patterns,memsim}.hpp.
tests/cpp/test_costmodel.cpp re-runs the reference's own cases
(test_exec_model.cpp, test_memsim.cpp, acceptance criterion 5); here its
account_tiled / account_levelwise are compared counter for counter with the
reference compiled from its headers (oracle/_ref) over a sweep of plans.
The GPU-side check that traced fft_tiled / fft_levelwise runs equal these
figures (criteria 4 and 7) is in tests/cpp/test_dropin.cpp.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "test_costmodel")


@pytest.fixture(scope="module")
def model_bin():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), BIN], check=True)
    return BIN


def test_reference_cost_model_cases(model_bin):
    r = subprocess.run([model_bin], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


CASES = [(2, 1024), (16, 4), (16, 1024), (256, 16), (1024, 1024), (4096, 64), (4096, 1024), (8192, 128),
         (65536, 1024), (65536, 16), (1 << 18, 512), (1 << 20, 1024)]


@pytest.mark.parametrize("n,cap", CASES)
def test_accounting_equals_reference(model_bin, reference, n, cap):
    out = subprocess.run([model_bin, "dump", str(n), str(cap)], capture_output=True, text=True, check=True).stdout
    tiled, level = ([int(v) for v in line.split()] for line in out.strip().splitlines())
    assert tiled == reference.account_tiled(n, cap)
    assert level == reference.account_levelwise(n)


@pytest.mark.parametrize("n,cap", [(16, 4), (4096, 64), (65536, 1024)])
def test_c_abi_accounting_equals_reference(reference, n, cap):
    """tilefft_account (the product library's cost model, used by the Python
    mirror and suite.py) against the reference."""
    import paper_1707_07263_b200 as tf
    from paper_1707_07263_b200 import _capi
    got = tf.tilefft.account_tiled(tf.make_plan(n, cap))
    assert [got[k] for k in _capi.ACCESS_STATS_FIELDS] == reference.account_tiled(n, cap)
    lw = tf.tilefft.account_levelwise(n)
    assert [lw[k] for k in _capi.ACCESS_STATS_FIELDS] == reference.account_levelwise(n)
    assert tf.tilefft.reduction_ratio(n, tf.make_plan(n, cap)) == tf.log2_exact(n) / tf.make_plan(n, cap).pass_count()
