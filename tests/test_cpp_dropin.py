"""The C++ drop-in headers (include/tilefft/*.hpp): they compile against the
C ABI (CPU) and pass the reference's own test cases on the B200 (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                   check=True)
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return os.path.join(CPP, "bin", "test_dropin")


def test_dropin_headers_compile():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu():
    r = subprocess.run([build()], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
