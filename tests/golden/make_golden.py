#!/usr/bin/env python3
"""Generate tests/golden/reference_fixtures.json from the REFERENCE itself.

Runs only where /root/reference exists (it builds oracle/_ref from the
reference headers). The JSON pins:
  * the golden vectors the reference's own tests hold (cited file:line);
  * make_plan geometry for a grid of (n, cap) (stage_plan.hpp:74-127);
  * exchange/interleave maps for the worked examples (test_stage_plan.cpp);
  * sha256 of fft_tiled / ifft_tiled / fft_levelwise outputs (fp32 and fp64)
    on random_bench_signal inputs, computed by the reference, for sizes up to
    2^20 — the GPU exact mode and the oracle must reproduce these bit for bit;
  * random_bench_signal prefixes and twiddle-table hashes.
"""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle_lib import Reference
    R = Reference()
    fx = {"generator": "tests/golden/make_golden.py (reference headers compiled via oracle/Makefile)"}

    # -- pinned vectors from the reference's tests --------------------------------------------
    x8 = np.array([1 + 1j, 2 - 1j, 0, -1 + 2j, 3, -2j, -2 + 1j, 1], dtype=np.complex128)
    fx["dft_len8"] = {"cite": "tests/test_reference_dft.cpp:65-79",
                      "x": [[v.real, v.imag] for v in x8],
                      "expected": [[4.0, 1.0], [1.9497474683058327, -1.7071067811865475], [1.0, -2.0],
                                   [-1.7071067811865475, 3.7071067811865475], [0.0, 3.0],
                                   [-7.949747468305833, -0.2928932188134524], [11.0, 2.0],
                                   [-0.2928932188134524, 2.2928932188134525]],
                      "reference_output": [[v.real, v.imag] for v in R.dft(x8)]}
    x2 = np.array([1.5 - 0.5j, 0.25 + 2.0j])
    fx["levelwise_n2"] = {"cite": "tests/test_fft_baseline.cpp:66-72", "x": [[1.5, -0.5], [0.25, 2.0]],
                          "expected": [[1.75, 1.5], [1.25, -2.5]],
                          "reference_output": [[v.real, v.imag] for v in R.fft_levelwise(x2, 16)]}
    fx["bit_reverse_8"] = {"cite": "tests/test_fft_baseline.cpp:57-64", "expected": [0, 4, 2, 6, 1, 5, 3, 7]}
    fx["exchange_16_4_stage1"] = {"cite": "tests/test_stage_plan.cpp:157-167",
                                  "expected": [int(R.lib.ref_exchange_index_map(16, 4, 1, q)) for q in range(16)]}
    fx["exchange_8_4_stage2"] = {"cite": "tests/test_stage_plan.cpp:169-180",
                                 "expected": [int(R.lib.ref_exchange_index_map(8, 4, 2, q)) for q in range(8)]}
    fx["gather_16_4"] = {"cite": "tests/test_stage_plan.cpp:142-155",
                         "stage1": [[int(R.lib.ref_gather_source_index(16, 4, 1, r, c)) for c in range(4)]
                                    for r in range(4)],
                         "stage2_0_2": int(R.lib.ref_gather_source_index(16, 4, 2, 0, 2)),
                         "stage2_3_1": int(R.lib.ref_gather_source_index(16, 4, 2, 3, 1))}
    ramp = np.arange(8, dtype=np.float64).astype(np.complex128)
    fx["exchange_transpose_8_4"] = {"cite": "tests/test_tiled_fft.cpp:168-175",
                                    "expected": [v.real for v in R.exchange_transpose(ramp, 4, 2)]}
    tw16 = R.twiddle(16, np.complex128)
    fx["interstage_minus_i"] = {"cite": "tests/test_tiled_fft.cpp:112-134",
                                "note": "plan (4,2): row 1, col 1 root W_4^1 = table16[4]",
                                "value": [tw16[4].real, tw16[4].imag]}

    # -- plans ----------------------------------------------------------------------------------
    plans = []
    for bits in range(1, 31):
        for cap_bits in (1, 2, 3, 4, 5, 10, 13):
            n, cap = 1 << bits, 1 << cap_bits
            if bits > 20 and cap_bits < 10:
                continue
            p = R.make_plan(n, cap)
            plans.append({"n": n, "cap": cap, **p})
    fx["plans"] = {"cite": "stage_plan.hpp:74-127; tests/test_stage_plan.cpp:26-128", "cases": plans}

    # -- twiddle tables --------------------------------------------------------------------------
    fx["twiddle_sha256"] = {str(res): {"f32": sha(R.twiddle(res, np.complex64)), "f64": sha(R.twiddle(res, np.complex128))}
                            for res in (2, 4, 8, 16, 64, 1024, 1 << 16, 1 << 20)}
    tw8 = R.twiddle(8, np.complex128)
    fx["twiddle_8"] = {"cite": "tests/test_twiddle.cpp:33-41", "values": [[v.real, v.imag] for v in tw8]}

    # -- inputs -----------------------------------------------------------------------------------
    fx["random_bench_signal"] = {"cite": "bench.hpp:128-138",
                                 "n16_seed1": [[v.real, v.imag] for v in R.random_bench_signal(16, 1)],
                                 "sha256_n1M_seed1": sha(R.random_bench_signal(1 << 20, 1))}

    # -- transform outputs (sha256 of the exact bytes) -----------------------------------------
    cases = []
    grid = [(2, 1024), (4, 2), (8, 4), (16, 4), (32, 2), (64, 4), (64, 8), (256, 16), (512, 8), (1024, 4),
            (1024, 32), (1024, 1024), (4096, 64), (8192, 1024), (1 << 16, 1024), (1 << 16, 256), (1 << 20, 1024),
            (1 << 20, 64)]
    for n, cap in grid:
        x = R.random_bench_signal(n, 1)
        for dt, tag in ((np.complex64, "f32"), (np.complex128, "f64")):
            xi = x.astype(dt)
            cases.append({"n": n, "cap": cap, "dtype": tag, "op": "fft_tiled", "sha256": sha(R.fft_tiled(xi, cap))})
            if n <= 1 << 16:
                cases.append({"n": n, "cap": cap, "dtype": tag, "op": "ifft_tiled",
                              "sha256": sha(R.fft_tiled(xi, cap, inverse=True))})
        if n <= 64:
            y = R.fft_tiled(x.astype(np.complex64), cap)
            cases.append({"n": n, "cap": cap, "dtype": "f32", "op": "fft_tiled_values",
                          "values": [[float(v.real), float(v.imag)] for v in y]})
    for n in (2, 8, 256, 4096):
        x = R.random_bench_signal(n, 1)
        cases.append({"n": n, "dtype": "f64", "op": "fft_levelwise", "sha256": sha(R.fft_levelwise(x))})
        cases.append({"n": n, "dtype": "f64", "op": "dft_reference", "sha256": sha(R.dft(x))})
    fx["transforms"] = {"cite": "tiled_fft.hpp:321-423, fft_baseline.hpp:66-116, reference_dft.hpp:41-77; "
                                "input random_bench_signal(n, seed=1) cast to the dtype, table resolution n",
                        "cases": cases}
    out = os.path.join(HERE, "reference_fixtures.json")
    with open(out, "w") as f:
        json.dump(fx, f, indent=1)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
