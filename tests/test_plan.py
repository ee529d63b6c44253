"""Host logic of the Python mirror (make_plan, index maps, twiddle table
construction) against the reference-generated fixtures and the reference's
own plan tests (test_stage_plan.cpp, test_twiddle.cpp). CPU only."""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import paper_1707_07263_b200 as tf

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = json.load(open(os.path.join(HERE, "golden", "reference_fixtures.json")))


def test_make_plan_matches_reference_for_all_fixture_cases():
    for c in FIX["plans"]["cases"]:
        p = tf.make_plan(c["n"], c["cap"])
        assert list(p.factors) == c["factors"]
        assert [[g.fft_len, g.levels, g.rows, g.sub_len, g.rows_per_sub, g.padded_stride, g.rows_per_tile,
                 g.tile_count] for g in p.stages] == c["geom"]
        assert list(p.sub_weights) == c["sub_weights"]
        assert list(p.out_weights) == c["out_weights"]


def test_make_plan_reference_cases():
    # test_stage_plan.cpp:26-107
    p = tf.make_plan(1024, 1024)
    assert p.factors == (1024,) and p.stage(1).padded_stride == 1025 and p.stage(1).tile_count == 1
    p = tf.make_plan(65536, 1024)
    assert p.factors == (256, 256) and p.stage(1).rows_per_tile == 4 and p.stage(1).tile_count == 64
    assert tf.make_plan(2048, 1024).factors == (64, 32)
    assert tf.make_plan(8192, 1024).factors == (128, 64)
    p = tf.make_plan(64, 4)
    assert p.factors == (4, 4, 4) and p.sub_weights == (4, 1) and p.out_weights == (1, 4, 16)
    assert p.stage(1).padded_stride == 4


def test_make_plan_errors():
    for args in [(0,), (1,), (48,), (1024, 0), (1024, 1), (1024, 100)]:
        with pytest.raises(ValueError):
            tf.make_plan(*args)
    p = tf.make_plan(16, 4)
    with pytest.raises(ValueError, match="pass out of range"):
        p.stage(0)
    with pytest.raises(ValueError):
        p.stage(3)
    with pytest.raises(ValueError):
        tf.make_plan(16, 4, tf.ExecConfig(warp_size=32, half_warp_size=8))


def test_index_maps_match_fixtures():
    p16 = tf.make_plan(16, 4)
    assert [tf.exchange_index_map(p16, 1, q) for q in range(16)] == FIX["exchange_16_4_stage1"]["expected"]
    p8 = tf.make_plan(8, 4)
    assert [tf.exchange_index_map(p8, 2, q) for q in range(8)] == FIX["exchange_8_4_stage2"]["expected"]
    g = FIX["gather_16_4"]
    assert [[tf.gather_source_index(p16.stage(1), r, c) for c in range(4)] for r in range(4)] == g["stage1"]
    assert tf.gather_source_index(p16.stage(2), 0, 2) == g["stage2_0_2"]
    assert tf.gather_source_index(p16.stage(2), 3, 1) == g["stage2_3_1"]
    assert tf.bit_reverse_permutation(8) == FIX["bit_reverse_8"]["expected"]


def test_exchange_maps_are_permutations():
    # test_stage_plan.cpp:182-196, :198-208
    for n, cap in [(64, 4), (256, 16), (4096, 64)]:
        p = tf.make_plan(n, cap)
        for s in range(1, p.pass_count() + 1):
            assert sorted(tf.exchange_index_map(p, s, q) for q in range(n)) == list(range(n))
            g = p.stage(s)
            for grow in range(0, g.rows, max(1, g.rows // 7)):
                for k in range(g.fft_len):
                    assert tf.scatter_target_index(p, s, grow, k) == tf.exchange_index_map(p, s, grow * g.fft_len + k)
    p = tf.make_plan(32, 32)
    assert [tf.final_output_index(p, 0, k) for k in range(32)] == list(range(32))


def test_twiddle_table_bit_identical_to_reference():
    # the Python API builds its table through the product library's host code
    pytest.importorskip("ctypes")
    try:
        tf._capi.load()
    except ImportError:
        pytest.skip("libtilefft_b200.so not built")
    for res, h in FIX["twiddle_sha256"].items():
        for dt, key in ((np.complex64, "f32"), (np.complex128, "f64")):
            t = tf.build_twiddle_table(int(res), dt)
            assert hashlib.sha256(t.values.tobytes()).hexdigest() == h[key], (res, key)


def test_twiddle_identities_exact():
    # test_twiddle.cpp:86-138; acceptance_main.cpp:120-156 (reduced sample)
    try:
        tf._capi.load()
    except ImportError:
        pytest.skip("libtilefft_b200.so not built")
    table = tf.build_twiddle_table(65536, np.complex128)
    rng = random.Random(0x7D11E5)
    for _ in range(2000):
        nb = rng.randint(1, 16)
        n = 1 << nb
        e = rng.randint(-(1 << 40), 1 << 40)
        m = 1 << rng.randint(0, 16 - nb)
        w = tf.twiddle_lookup(table, n, e)
        assert tf.twiddle_lookup(table, n, e + n) == w
        cw = tf.twiddle_lookup(table, n, -e)
        assert cw.real == w.real and cw.imag == -w.imag
        assert tf.twiddle_lookup(table, m * n, m * e) == w


def test_twiddle_errors():
    for r in (0, 1, 24):
        with pytest.raises(ValueError, match="resolution must be a power of two"):
            tf.build_twiddle_table(r)
