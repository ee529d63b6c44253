"""Report harness (paper_1707_07263_b200/suite.py): the reference's run_suite
schema (bench.hpp:70-110, 87-89) with GPU rows and a cuFFT comparison column."""
import numpy as np
import pytest

from paper_1707_07263_b200 import suite


def test_csv_header_extends_reference_schema():
    # bench.hpp:87-89, pinned by test_bench.cpp:148-156
    assert suite.kCsvHeader == ("size,algorithm,passes,max_err_vs_oracle,slow_elem_accesses,slow_transactions,"
                                "bank_conflict_cycles,barriers,wall_time_ns,repetitions")
    assert suite.kCsvHeaderB200.startswith(suite.kCsvHeader + ",")
    assert suite.table1_sizes() == [16, 64, 256, 1024, 4096, 16384, 65536]


def test_render_parse_roundtrip():
    rows = [suite.BenchRow(16, "oracle", 0, 0.0, repetitions=3, wall_time_ns=5),
            suite.BenchRow(16, "b200", 1, 1.5e-15, 32, 0, 0, 1, 123, 3, 4567, 1.25, 2.5),
            suite.BenchRow(1 << 26, "b200", 3, None, 3 << 27, 0, 0, 3, 9, 3, 10, 3.0, 4.0)]
    for fmt in ("csv", "json"):
        text = suite.render_report(rows, fmt)
        back = suite.parse_report(text, fmt)
        assert [(r.size, r.algorithm, r.passes, r.max_err_vs_oracle, r.device_time_ns) for r in back] == \
               [(r.size, r.algorithm, r.passes, r.max_err_vs_oracle, r.device_time_ns) for r in rows]
    assert suite.render_report(rows, "csv").splitlines()[0] == suite.kCsvHeaderB200


def test_signal_is_deterministic_uniform():
    a = suite.suite_signal(4096, 1)
    assert np.array_equal(a, suite.suite_signal(4096, 1))
    assert not np.array_equal(a, suite.suite_signal(4096, 2))
    assert np.all(np.abs(a.real) <= 1) and np.all(np.abs(a.imag) <= 1)
    assert abs(a.real.mean()) < 0.05 and 0.3 < a.real.std() < 0.65


def test_size_validation_matches_reference_message():
    with pytest.raises(ValueError, match="is not a power of two"):
        suite.run_suite([12])
    with pytest.raises(ValueError, match="no sizes given"):
        suite.run_suite([])


def test_direct_dft_matches_numpy():
    x = suite.suite_signal(64, 3)
    assert np.max(np.abs(suite._direct_dft(x) - np.fft.fft(x))) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_run_suite_gpu_rows(dtype):
    rows = []
    got = suite.run_suite([16, 1024, 1 << 16], suite.SuiteOptions(repetitions=2, dtype=dtype, on_row=rows.append))
    assert got == rows
    algs = [(r.size, r.algorithm) for r in got]
    assert algs[:5] == [(16, a) for a in suite.ALGORITHMS]
    assert (1 << 16, "oracle") not in algs and (1 << 16, "b200") in algs
    tol = 1e-9 if dtype == np.complex128 else 1e-3
    for r in got:
        if r.max_err_vs_oracle is not None:
            assert r.max_err_vs_oracle <= tol * r.size * 1.5
        if r.algorithm in ("b200", "tiled", "levelwise"):
            assert r.device_time_ns > 0 and r.slow_elem_accesses == 2 * r.size * r.passes
