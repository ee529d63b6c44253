"""bench.py contract pieces that run without a GPU: the reference arm's JSON line (the reference's own
fft_tiled on host cores), the config object both arms share, and the synthetic input generator."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def test_splitmix_input_matches_the_oracle():
    import bench
    from oracle_lib import Oracle
    got = bench.splitmix_signal(4096, seed=3)
    want = Oracle().splitmix_signal(4096, 3)
    assert got.dtype == np.complex64
    assert np.array_equal(got.view(np.uint32), np.asarray(want, np.complex64).view(np.uint32))


def test_config_keys_are_identical_for_both_arms():
    import bench
    for name in bench.CONFIGS:
        k = bench.config_key(name)
        assert set(k) == {"workload", "name", "n", "batch_per_gpu", "kind", "l2"}
        assert k["name"] == name
    assert bench.DEVICE_FACTORS.keys() == bench.CONFIGS.keys()


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref")), reason="compiled reference absent")
def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1d_2e20",
                        "--steps", "2", "--warmup", "1", "--ref-budget", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"] == {"value": d["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    import bench
    assert d["config"] == bench.config_key("1d_2e20")
