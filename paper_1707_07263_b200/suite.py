"""Size-sweep report harness: the reference's ``run_suite`` (bench.hpp:170-291)
with GPU rows.

Same row schema and CSV header as the reference (``kCsvHeader``,
bench.hpp:87-89), extended with device columns, and the same validation rule
(a fast path that disagrees with its reference past tolerance raises
``BenchValidationError`` after the rows produced so far were delivered to
``on_row``, bench.hpp:93-96,185-190). Rows per size, in order:

  ``oracle``    direct O(N^2) DFT in fp64 (numpy; N <= oracle_max), the error reference
  ``levelwise`` the paper's previous method on the GPU (TILEFFT_MODE_LEVELWISE)
  ``tiled``     fft_tiled on the GPU, exact tier (bit-identical to the reference's)
  ``b200``      fft_tiled on the GPU, fast tier (the product path)
  ``cufft``     torch.fft.fft on the same device (comparison column only; the
                paper's CUFFT column, PAPER.md:217-235 — not on the product path)

Differences from the reference harness, on purpose: sizes up to 2^30 (the
reference caps at 2^20, bench.hpp:173-177); ``wall_time_ns`` is the
reference's best-of-R host-to-host time (vector in, vector out) and
``device_time_ns`` the best-of-R device-resident time (CUDA events);
``slow_elem_accesses`` / ``barriers`` follow the reference's 2 N p law for the
device passes actually run (memsim.hpp:59-63). ``slow_transactions`` /
``bank_conflict_cycles`` are the reference's cost model (memsim.hpp, through
``tilefft_account``) for the rows that execute the reference's algorithm
(``levelwise``, ``tiled``); the model does not describe the fast tier's
radix-32 kernels or cuFFT, so those rows carry -1 ("not modelled"), never a
misleading 0. The reference's CSV writer
prints the algorithm name twice (bench.hpp:303-304); this one prints it once.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import sys
import time
from typing import Callable, List, Optional

import numpy as np

from . import _capi
from . import tilefft as tf

kCsvHeader = ("size,algorithm,passes,max_err_vs_oracle,slow_elem_accesses,slow_transactions,"
              "bank_conflict_cycles,barriers,wall_time_ns,repetitions")
kCsvHeaderB200 = kCsvHeader + ",device_time_ns,gflops,hbm_gbs"

ALGORITHMS = ("oracle", "levelwise", "tiled", "b200", "cufft")


class BenchValidationError(RuntimeError):  # bench.hpp:93-96
    pass


@dataclasses.dataclass
class BenchRow:  # bench.hpp:70-83 + device columns
    size: int
    algorithm: str
    passes: int = 0
    max_err_vs_oracle: Optional[float] = None
    slow_elem_accesses: int = 0
    slow_transactions: int = 0
    bank_conflict_cycles: int = 0
    barriers: int = 0
    wall_time_ns: int = 0
    repetitions: int = 0
    device_time_ns: int = 0
    gflops: float = 0.0
    hbm_gbs: float = 0.0


@dataclasses.dataclass
class SuiteOptions:  # bench.hpp:98-110
    tile_capacity: int = 1024
    oracle_max: int = 8192
    repetitions: int = 9
    seed: int = 1
    threads: int = 1
    dtype: type = np.complex128
    include_cufft: bool = True
    exact_max: int = 1 << 22   # levelwise / exact-tier rows build an n-entry host root table
    device: int = 0
    on_row: Optional[Callable[[BenchRow], None]] = None


def table1_sizes() -> List[int]:  # bench.hpp:114-116
    return [16, 64, 256, 1024, 4096, 16384, 65536]


def suite_signal(n: int, seed: int) -> np.ndarray:
    """Per-size reproducible signal, uniform(-1, 1) re and im. Counter-based
    (splitmix64 of seed ^ golden * n and the index) so it is cheap at 2^30;
    the reference's mt19937_64 stream is what the parity tests use."""
    idx = np.arange(2 * n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = idx + np.uint64((seed ^ (0x9E3779B97F4A7C15 * n)) & 0xFFFFFFFFFFFFFFFF)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53)) * 2.0 - 1.0
    return (u[0::2] + 1j * u[1::2]).astype(np.complex128)


def _direct_dft(x: np.ndarray) -> np.ndarray:
    """O(N^2) DFT in fp64 with exact-angle roots (reference_dft.hpp:41-60)."""
    n = x.shape[-1]
    k = np.arange(n)
    out = np.empty(n, dtype=np.complex128)
    xd = x.astype(np.complex128)
    for j in range(n):
        out[j] = np.sum(xd * np.exp(-2j * np.pi * ((j * k) % n) / n))
    return out


def _max_abs_error(a: np.ndarray, b: np.ndarray) -> float:  # reference_dft.hpp:81-91
    return float(np.max(np.abs(a.astype(np.complex128) - b.astype(np.complex128)))) if a.size else 0.0


def _best_ns(reps: int, fn) -> int:  # bench.hpp:149-161
    best = None
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        fn()
        dt = max(time.perf_counter_ns() - t0, 1)
        best = dt if best is None else min(best, dt)
    return int(best)


def _device_best_ns(reps: int, fn, inner: int = 10) -> int:
    """Best-of-R device time per call, each sample `inner` back-to-back calls
    between two CUDA events on the launching stream (so host submission time
    of small transforms does not show up as device time)."""
    import torch
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(inner):
            fn()
        b.record()
        b.synchronize()
        dt = max(int(a.elapsed_time(b) * 1e6 / inner), 1)
        best = dt if best is None else min(best, dt)
    return int(best)


def run_suite(sizes: List[int], options: SuiteOptions = SuiteOptions()) -> List[BenchRow]:
    """bench.hpp:170-291 with GPU rows (see module docstring)."""
    import torch
    tf._require(len(sizes) > 0, "run_suite: no sizes given")
    for n in sizes:
        tf._require(tf.is_power_of_two(n) and 2 <= n <= (1 << 30),
                    f"run_suite: size {n} is not a power of two in [2, 1073741824]")
    tf._require(options.repetitions >= 1, "run_suite: repetitions must be >= 1")
    dt = np.dtype(options.dtype)
    tf._require(dt in (np.complex64, np.complex128), "run_suite: dtype must be complex64 or complex128")
    real_eps = 1e-9 if dt == np.complex128 else 1e-3
    rows: List[BenchRow] = []
    dev = torch.device("cuda", options.device)

    def push(row: BenchRow) -> None:
        rows.append(row)
        if options.on_row:
            options.on_row(row)

    for n in sizes:
        x = suite_signal(n, options.seed).astype(dt)
        amp = float(np.max(np.abs(x)))
        oracle_tol = real_eps * n * amp
        flops = 5.0 * n * math.log2(n)
        oracle_out = None
        if n <= options.oracle_max:
            holder = {}
            t = _best_ns(options.repetitions if n <= 1024 else 1, lambda: holder.setdefault("y", _direct_dft(x)))
            oracle_out = holder["y"]
            push(BenchRow(n, "oracle", 0, 0.0, repetitions=options.repetitions, wall_time_ns=t))

        def check(name: str, y: np.ndarray) -> Optional[float]:
            if oracle_out is None:
                return None
            err = _max_abs_error(y, oracle_out)
            if not err <= oracle_tol:
                raise BenchValidationError(f"{name} transform of size {n} deviates from the reference by "
                                           f"{err:.17g} (tolerance {oracle_tol:.17g})")
            return err

        xd = torch.from_numpy(x).to(dev)
        yd = torch.empty_like(xd)
        stream = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
        table = tf.build_twiddle_table(n, dt.type) if n <= options.exact_max else None
        plan = tf.make_plan(n, options.tile_capacity)

        # levelwise (the paper's previous method): log2 n sweeps + the bit reversal
        if table is not None:
            lw = tf._device_plan(n, 1, None, dt.itemsize, _capi.MODE_LEVELWISE, table, options.device)
            y = tf.fft_levelwise(x, table)
            levels = tf.log2_exact(n)
            wall = _best_ns(options.repetitions, lambda: tf.fft_levelwise(x, table))
            dev_ns = _device_best_ns(options.repetitions, lambda: lw.exec_device(xd.data_ptr(), yd.data_ptr(),
                                                                                   _capi.FORWARD, stream()))
            lwm = _capi.account(n, options.tile_capacity, _capi.ACCOUNT_LEVELWISE)
            push(BenchRow(n, "levelwise", levels, check("levelwise", y), 2 * n * levels, lwm["slow_transactions"],
                          lwm["bank_conflict_cycles"], levels, wall,
                          options.repetitions, dev_ns, flops / dev_ns, 2 * n * (levels + 1) * dt.itemsize / dev_ns))

            # tiled (exact tier): the reference's own plan and table, bit for bit
            ex = tf._device_plan(n, 1, plan.factors, dt.itemsize, _capi.MODE_EXACT, table, options.device)
            y = tf.fft_tiled(x, plan, table, mode="exact")
            p = plan.pass_count()
            wall = _best_ns(options.repetitions, lambda: tf.fft_tiled(x, plan, table, mode="exact"))
            dev_ns = _device_best_ns(options.repetitions, lambda: ex.exec_device(xd.data_ptr(), yd.data_ptr(),
                                                                                   _capi.FORWARD, stream()))
            tm = _capi.account(n, options.tile_capacity, _capi.ACCOUNT_TILED)
            push(BenchRow(n, "tiled", p, check("tiled", y), 2 * n * p, tm["slow_transactions"],
                          tm["bank_conflict_cycles"], p, wall, options.repetitions, dev_ns,
                          flops / dev_ns, 2 * n * p * dt.itemsize / dev_ns))

        # b200 (fast tier, the product path)
        fp = tf._device_plan(n, 1, plan.factors, dt.itemsize, _capi.MODE_FAST, None, options.device)
        y = tf.fft_tiled(x, plan)
        dp = fp.info()["passes"]
        wall = _best_ns(options.repetitions, lambda: tf.fft_tiled(x, plan))
        dev_ns = _device_best_ns(options.repetitions, lambda: fp.exec_device(xd.data_ptr(), yd.data_ptr(),
                                                                               _capi.FORWARD, stream()))
        push(BenchRow(n, "b200", dp, check("b200", y), 2 * n * dp, -1, -1, dp, wall, options.repetitions, dev_ns,
                      flops / dev_ns, 2 * n * dp * dt.itemsize / dev_ns))

        if options.include_cufft:
            y = torch.fft.fft(xd).cpu().numpy()
            wall = _best_ns(options.repetitions, lambda: torch.fft.fft(torch.from_numpy(x).to(dev)).cpu())
            dev_ns = _device_best_ns(options.repetitions, lambda: torch.fft.fft(xd))
            push(BenchRow(n, "cufft", 0, check("cufft", y), 0, -1, -1, 0, wall, options.repetitions, dev_ns,
                          flops / dev_ns, 0.0))
        del xd, yd
    return rows


def render_report(rows: List[BenchRow], fmt: str = "csv") -> str:  # bench.hpp:293-342
    if fmt == "csv":
        out = [kCsvHeaderB200]
        for r in rows:
            err = "" if r.max_err_vs_oracle is None else f"{r.max_err_vs_oracle:.17g}"
            out.append(f"{r.size},{r.algorithm},{r.passes},{err},{r.slow_elem_accesses},{r.slow_transactions},"
                       f"{r.bank_conflict_cycles},{r.barriers},{r.wall_time_ns},{r.repetitions},"
                       f"{r.device_time_ns},{r.gflops:.3f},{r.hbm_gbs:.3f}")
        return "\n".join(out) + "\n"
    tf._require(fmt == "json", "render_report: format must be csv or json")
    return json.dumps([dataclasses.asdict(r) for r in rows], indent=2) + "\n"


def parse_report(text: str, fmt: str = "csv") -> List[BenchRow]:
    if fmt == "json":
        return [BenchRow(**d) for d in json.loads(text)]
    lines = [ln for ln in text.splitlines() if ln]
    tf._require(lines and lines[0] == kCsvHeaderB200, "parse_report: unexpected CSV header")
    rows = []
    for ln in lines[1:]:
        c = ln.split(",")
        rows.append(BenchRow(int(c[0]), c[1], int(c[2]), float(c[3]) if c[3] else None, int(c[4]), int(c[5]),
                             int(c[6]), int(c[7]), int(c[8]), int(c[9]), int(c[10]), float(c[11]), float(c[12])))
    return rows


def main(argv=None) -> int:  # tools/tilefft_bench.cpp:57-153
    ap = argparse.ArgumentParser(description="tilefft B200 size sweep (reference run_suite schema + GPU columns)")
    ap.add_argument("--sizes", default=",".join(str(s) for s in table1_sizes()))
    ap.add_argument("--tile-capacity", type=int, default=1024)
    ap.add_argument("--oracle-max", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp64")
    ap.add_argument("--no-cufft", action="store_true")
    ap.add_argument("--format", choices=["csv", "json"], default="csv")
    ap.add_argument("--out", default="-")
    a = ap.parse_args(argv)
    sizes = []
    for tok in a.sizes.split(","):
        tok = tok.strip()
        sizes.append(1 << int(tok[2:]) if tok.startswith("2^") else int(tok))
    opts = SuiteOptions(tile_capacity=a.tile_capacity, oracle_max=a.oracle_max, repetitions=a.reps, seed=a.seed,
                        dtype=np.complex64 if a.precision == "fp32" else np.complex128,
                        include_cufft=not a.no_cufft,
                        on_row=lambda r: print(f"  {r.size:>10} {r.algorithm:<9} {r.device_time_ns:>12} ns",
                                               file=sys.stderr))
    rows: List[BenchRow] = []
    try:
        rows = run_suite(sizes, opts)
        rc = 0
    except BenchValidationError as e:  # partial report preserved (tools/tilefft_bench.cpp:126-136)
        print(f"validation failed: {e}", file=sys.stderr)
        rc = 1
    text = render_report(rows, a.format)
    if a.out == "-":
        sys.stdout.write(text)
    else:
        with open(a.out, "w") as f:
            f.write(text)
    return rc


if __name__ == "__main__":
    raise SystemExit(main())
