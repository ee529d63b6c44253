"""Pin the oracle (CPU restatement, oracle/tilefft_oracle.c) to the reference.

(a) against the golden vectors of the reference's own tests and the
    reference-generated fixtures in tests/golden/reference_fixtures.json
    (made by tests/golden/make_golden.py from the compiled reference);
(b) against the compiled reference itself (oracle/_ref), when present.
CPU only.
"""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = json.load(open(os.path.join(HERE, "golden", "reference_fixtures.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cplx(pairs, dtype=np.complex128):
    return np.array([complex(a, b) for a, b in pairs], dtype=dtype)


def test_golden_len8_spectrum(oracle):
    f = FIX["dft_len8"]
    got = oracle.dft(cplx(f["x"]))
    assert np.max(np.abs(got - cplx(f["expected"]))) < 1e-13  # test_reference_dft.cpp:65-79 tolerance
    assert np.array_equal(got, cplx(f["reference_output"]))


def test_exact_n2_butterfly(oracle):
    f = FIX["levelwise_n2"]
    got = oracle.fft_levelwise(cplx(f["x"]), res=16)
    assert np.array_equal(got, cplx(f["expected"]))


def test_bit_reverse_table(oracle):
    assert [int(oracle.lib.orc_bit_reverse(i, 3)) for i in range(8)] == FIX["bit_reverse_8"]["expected"]


def test_exchange_and_gather_maps(oracle):
    p16 = oracle.make_plan(16, 4)
    assert [int(oracle.lib.orc_exchange_index_map(p16, 1, q)) for q in range(16)] == \
        FIX["exchange_16_4_stage1"]["expected"]
    p8 = oracle.make_plan(8, 4)
    assert [int(oracle.lib.orc_exchange_index_map(p8, 2, q)) for q in range(8)] == FIX["exchange_8_4_stage2"]["expected"]
    g = FIX["gather_16_4"]
    assert [[int(oracle.lib.orc_gather_source_index(p16, 1, r, c)) for c in range(4)] for r in range(4)] == g["stage1"]
    assert int(oracle.lib.orc_gather_source_index(p16, 2, 0, 2)) == g["stage2_0_2"]
    assert int(oracle.lib.orc_gather_source_index(p16, 2, 3, 1)) == g["stage2_3_1"]


def test_interstage_minus_i(oracle):
    t = oracle.twiddle(16, np.complex128)
    assert [t[4].real, t[4].imag] == FIX["interstage_minus_i"]["value"] == [0.0, -1.0]


def test_plans_match_reference_geometry(oracle):
    for c in FIX["plans"]["cases"]:
        p = oracle.make_plan(c["n"], c["cap"])
        assert oracle.factors(p) == c["factors"], c
        geom = [[getattr(p.stages[s], k) for k in ("fft_len", "levels", "rows", "sub_len", "rows_per_sub",
                                                   "padded_stride", "rows_per_tile", "tile_count")]
                for s in range(p.passes)]
        assert geom == c["geom"]
        assert [p.sub_weights[i] for i in range(p.passes - 1)] == c["sub_weights"]
        assert [p.out_weights[i] for i in range(p.passes)] == c["out_weights"]


def test_plan_rejects_bad_shapes(oracle):
    for n, cap in [(0, 1024), (1, 1024), (48, 1024), (1024, 0), (1024, 1), (1024, 100)]:
        with pytest.raises(ValueError):
            oracle.make_plan(n, cap)


def test_twiddle_tables_bit_identical(oracle):
    for res, h in FIX["twiddle_sha256"].items():
        assert sha(oracle.twiddle(int(res), np.complex64)) == h["f32"], res
        assert sha(oracle.twiddle(int(res), np.complex128)) == h["f64"], res
    t8 = oracle.twiddle(8, np.complex128)
    assert np.array_equal(t8, cplx(FIX["twiddle_8"]["values"]))


def test_random_bench_signal(oracle):
    f = FIX["random_bench_signal"]
    assert np.array_equal(oracle.random_bench_signal(16, 1), cplx(f["n16_seed1"]))
    assert sha(oracle.random_bench_signal(1 << 20, 1)) == f["sha256_n1M_seed1"]


@pytest.mark.parametrize("case", [c for c in FIX["transforms"]["cases"]], ids=lambda c: f"{c['op']}-{c['n']}-"
                         f"{c.get('cap', '')}-{c['dtype']}")
def test_transforms_bit_identical_to_reference(oracle, case):
    n = case["n"]
    dt = np.complex64 if case["dtype"] == "f32" else np.complex128
    x = oracle.random_bench_signal(n, 1).astype(dt)
    op = case["op"]
    if op == "fft_tiled":
        got = oracle.fft_tiled(x, case["cap"])
    elif op == "ifft_tiled":
        got = oracle.fft_tiled(x, case["cap"], inverse=True)
    elif op == "fft_tiled_values":
        assert np.array_equal(oracle.fft_tiled(x, case["cap"]), cplx(case["values"], np.complex64))
        return
    elif op == "fft_levelwise":
        got = oracle.fft_levelwise(x)
    else:
        got = oracle.dft(x)
    assert sha(got) == case["sha256"]


def test_tiled_single_pass_equals_levelwise(oracle):
    # test_tiled_fft.cpp:226-234: p = 1 tiled is bit-identical to levelwise
    x = oracle.random_signal(256, 41)
    assert np.array_equal(oracle.fft_tiled(x, 1024), oracle.fft_levelwise(x))


def test_oracle_sweep_against_dft(oracle):
    # acceptance_main.cpp:69-98 (reduced: 3 signals per size)
    for bits in range(1, 13):
        n = 1 << bits
        for sig in range(3):
            x = oracle.random_signal(n, 0xACCE9700 + 1000003 * n + sig)
            tol = 1e-9 * n * np.max(np.abs(x))
            ref = oracle.dft(x)
            assert np.max(np.abs(oracle.fft_tiled(x) - ref)) <= tol
            assert np.max(np.abs(oracle.fft_levelwise(x) - ref)) <= tol


def test_oracle_matches_compiled_reference(oracle, reference):
    for n, cap in [(2, 1024), (64, 4), (4096, 64), (1 << 16, 1024), (1 << 18, 512)]:
        for dt in (np.complex64, np.complex128):
            x = oracle.random_bench_signal(n, 7).astype(dt)
            assert np.array_equal(oracle.fft_tiled(x, cap), reference.fft_tiled(x, cap))
            assert np.array_equal(oracle.fft_tiled(x, cap, inverse=True), reference.fft_tiled(x, cap, inverse=True))


def test_permute_matches_exchange_composition(oracle):
    # permute-only tiled pass == gather(bitrev) then scatter maps of every pass
    for n, cap in [(16, 4), (64, 4), (256, 16), (4096, 64)]:
        ramp = np.arange(n, dtype=np.float32).astype(np.complex64)
        got = oracle.permute_tiled(ramp, cap).real.astype(np.int64)
        p = oracle.make_plan(n, cap)
        cur = np.arange(n)
        for s in range(1, p.passes + 1):
            g = p.stages[s - 1]
            nxt = np.empty(n, np.int64)
            L, rps = g.fft_len, g.rows_per_sub
            for grow in range(g.rows):
                for c in range(L):
                    src = oracle.lib.orc_gather_source_index(p, s, grow, int(oracle.lib.orc_bit_reverse(c, g.levels)))
                    dst = oracle.lib.orc_exchange_index_map(p, s, grow * L + c)
                    nxt[dst] = cur[src]
            cur = nxt
        assert np.array_equal(got, cur)
