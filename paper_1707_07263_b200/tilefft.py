"""Python mirror of the reference's plan/execute API, executed on the B200.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/tilefft (``make_plan`` stage_plan.hpp:74-127,
``build_twiddle_table`` twiddle.hpp:47-73, ``fft_tiled`` tiled_fft.hpp:321-407,
``ifft_tiled`` :410-423, the index maps stage_plan.hpp:135-179): invalid
arguments raise ``ValueError`` where the reference throws
``std::invalid_argument``. The plan is host logic (as in the reference); every
transform runs through the C ABI (include/tilefft_b200.h) on the GPU — there is
no CPU execution path.

Complex data is numpy ``complex64`` (Real=float) or ``complex128``
(Real=double), the memory layout of ``std::vector<std::complex<Real>>``.
"""
from __future__ import annotations

import collections
import dataclasses
import hashlib
import os
import threading
from typing import List, Optional

import numpy as np

from . import _capi

kPi = 3.141592653589793238462643383279502884
kDefaultTwiddleResolution = 1 << 20  # twiddle.hpp:27


def is_power_of_two(v: int) -> bool:  # common.hpp:36-38
    return v > 0 and (v & (v - 1)) == 0


def log2_exact(v: int) -> int:  # common.hpp:41-43
    return (v & -v).bit_length() - 1


def _require(cond: bool, msg: str) -> None:  # common.hpp:47-51
    if not cond:
        raise ValueError(msg)


def bit_reverse(value: int, bits: int) -> int:  # common.hpp:54-60
    out = 0
    for i in range(bits):
        out = (out << 1) | ((value >> i) & 1)
    return out


@dataclasses.dataclass(frozen=True)
class ExecConfig:  # exec_model.hpp:33-53 (only bank_count reaches the plan)
    warp_size: int = 32
    half_warp_size: int = 16
    bank_count: int = 16
    word_bytes: int = 8
    segment_bytes: int = 128

    def element_bytes(self) -> int:
        return 2 * self.word_bytes

    def validate(self) -> None:
        _require(all(is_power_of_two(v) for v in (self.warp_size, self.half_warp_size, self.bank_count,
                                                  self.word_bytes, self.segment_bytes)),
                 "ExecConfig: all parameters must be powers of two")
        _require(self.warp_size == 2 * self.half_warp_size, "ExecConfig: warp_size must be twice half_warp_size")
        _require(self.segment_bytes >= self.element_bytes(), "ExecConfig: a segment must hold at least one element")


@dataclasses.dataclass(frozen=True)
class StageGeometry:  # stage_plan.hpp:36-45
    fft_len: int
    levels: int
    rows: int
    sub_len: int
    rows_per_sub: int
    padded_stride: int
    rows_per_tile: int
    tile_count: int


@dataclasses.dataclass(frozen=True)
class StagePlan:  # stage_plan.hpp:49-69
    n_total: int
    tile_capacity: int
    bank_count: int
    factors: tuple
    stages: tuple
    sub_weights: tuple
    out_weights: tuple

    def pass_count(self) -> int:
        return len(self.factors)

    def stage(self, p: int) -> StageGeometry:
        _require(1 <= p <= len(self.stages), "StagePlan::stage: pass out of range")
        return self.stages[p - 1]


def make_plan(n: int, tile_capacity: int = 1024, config: ExecConfig = ExecConfig()) -> StagePlan:
    """stage_plan.hpp:74-127."""
    _require(is_power_of_two(n) and n >= 2, "make_plan: n must be a power of two >= 2")
    _require(is_power_of_two(tile_capacity) and tile_capacity >= 2,
             "make_plan: tile_capacity must be a power of two >= 2")
    config.validate()
    total_bits, cap_bits = log2_exact(n), log2_exact(tile_capacity)
    passes = (total_bits + cap_bits - 1) // cap_bits
    base_bits, extra = total_bits // passes, total_bits % passes
    factors = [1 << (base_bits + (1 if s < extra else 0)) for s in range(passes)]
    stages = []
    sub_len = n
    for s in range(passes):
        L = factors[s]
        rows = n // L
        rps = sub_len // L
        rpt = min(rows, tile_capacity // L)
        stages.append(StageGeometry(L, log2_exact(L), rows, sub_len, rps,
                                    L + (1 if L % config.bank_count == 0 else 0), rpt, rows // rpt))
        sub_len = rps
    out_w = [1] * passes
    for i in range(1, passes):
        out_w[i] = out_w[i - 1] * factors[i - 1]
    sub_w = [1] * (passes - 1)
    for i in range(passes - 2, -1, -1):
        sub_w[i] = sub_w[i + 1] * factors[i + 1] if i + 1 < passes - 1 else 1
    return StagePlan(n, tile_capacity, config.bank_count, tuple(factors), tuple(stages), tuple(sub_w), tuple(out_w))


# ---- index maps (host logic, stage_plan.hpp:135-179) ---------------------------------------------
def gather_source_index(geom: StageGeometry, grow: int, col: int) -> int:
    return (grow // geom.rows_per_sub) * geom.sub_len + grow % geom.rows_per_sub + col * geom.rows_per_sub


def final_output_index(plan: StagePlan, sub: int, k: int) -> int:
    p = plan.pass_count()
    out, rem = k * plan.out_weights[p - 1], sub
    for i in range(p - 1):
        digit, rem = divmod(rem, plan.sub_weights[i])
        out += digit * plan.out_weights[i]
    return out


def exchange_index_map(plan: StagePlan, stage: int, q: int) -> int:
    geom = plan.stage(stage)
    if stage < plan.pass_count():
        sub, local = divmod(q, geom.sub_len)
        r, k = divmod(local, geom.fft_len)
        return sub * geom.sub_len + k * geom.rows_per_sub + r
    return final_output_index(plan, q // geom.fft_len, q % geom.fft_len)


def scatter_target_index(plan: StagePlan, stage: int, grow: int, k: int) -> int:
    return exchange_index_map(plan, stage, grow * plan.stage(stage).fft_len + k)


def bit_reverse_permutation(n: int) -> List[int]:  # fft_baseline.hpp:39-47
    _require(is_power_of_two(n), "bit_reverse_permutation: n must be a power of two")
    bits = log2_exact(n)
    return [bit_reverse(i, bits) for i in range(n)]


# ---- twiddle table --------------------------------------------------------------------------------
@dataclasses.dataclass
class TwiddleTable:  # twiddle.hpp:40-44
    resolution: int
    values: np.ndarray  # complex64 / complex128, length resolution


def build_twiddle_table(resolution: int = kDefaultTwiddleResolution, dtype=np.complex128) -> TwiddleTable:
    """twiddle.hpp:47-73 — values bit-identical to the reference's table."""
    _require(is_power_of_two(resolution) and resolution >= 2,
             "build_twiddle_table: resolution must be a power of two >= 2")
    dtype = np.dtype(dtype)
    _require(dtype in (np.dtype(np.complex64), np.dtype(np.complex128)), "build_twiddle_table: dtype")
    vals = np.empty(resolution, dtype=dtype)
    _capi.build_twiddle(resolution, dtype.itemsize, vals.ctypes.data)
    return TwiddleTable(resolution, vals)


def twiddle_lookup(table: TwiddleTable, n: int, e: int):  # twiddle.hpp:79-91
    _require(is_power_of_two(n), "twiddle_lookup: n must be a power of two")
    _require(table.resolution != 0 and n <= table.resolution and table.resolution % n == 0,
             "twiddle_lookup: n must divide the table resolution")
    return table.values[(e % n) * (table.resolution // n)]


# ---- cost model (memsim.hpp / access_patterns.hpp, host logic) -------------------------------------
def account_tiled(plan: StagePlan) -> dict:
    """memsim.hpp:58-95: the reference's closed-form AccessStats of fft_tiled under `plan`."""
    _require(plan.pass_count() >= 1, "account_tiled: empty plan")
    _require(plan.bank_count == ExecConfig().bank_count, "account_tiled: plan was built for a different bank count")
    return _capi.account(plan.n_total, plan.tile_capacity, _capi.ACCOUNT_TILED)


def account_levelwise(n: int) -> dict:
    """memsim.hpp:38-55: AccessStats of fft_levelwise (the reorder sweep excluded)."""
    _require(is_power_of_two(n) and n >= 2, "account_levelwise: n must be a power of two >= 2")
    return _capi.account(n, 2, _capi.ACCOUNT_LEVELWISE)


def reduction_ratio(n: int, plan: StagePlan) -> float:
    """memsim.hpp:99-104."""
    _require(n == plan.n_total, "reduction_ratio: n does not match the plan")
    _require(plan.pass_count() >= 1, "reduction_ratio: empty plan")
    return log2_exact(n) / plan.pass_count()


# ---- execution ------------------------------------------------------------------------------------
_plan_cache: "collections.OrderedDict" = collections.OrderedDict()
_cache_lock = threading.Lock()
# Each cached plan pins device workspace and host staging: least recently
# used plans are released beyond this many entries.
PLAN_CACHE_CAPACITY = int(os.environ.get("TILEFFT_PLAN_CACHE", "16"))


def _cached_plan(key, create):
    with _cache_lock:
        p = _plan_cache.get(key)
        if p is None:
            p = create()
            _plan_cache[key] = p
            while len(_plan_cache) > max(1, PLAN_CACHE_CAPACITY):
                _plan_cache.popitem(last=False)  # released when its last user drops it (DevicePlan.__del__)
        else:
            _plan_cache.move_to_end(key)
        return p


def _device_plan(n, batch, factors, elem_bytes, mode, table, device):
    uses_table = table is not None and mode in (_capi.MODE_EXACT, _capi.MODE_LEVELWISE)
    # FAST plans choose their own device passes: keyed by shape only. Table
    # plans copy the roots they use at creation: keyed by those roots' bytes.
    fp = None
    if uses_table:
        roots = table.values[:: table.resolution // n][:n]
        fp = (table.resolution, hashlib.blake2b(np.ascontiguousarray(roots).tobytes(), digest_size=16).hexdigest())
    key = (n, batch, tuple(factors) if (factors and mode != _capi.MODE_FAST) else None, elem_bytes, mode, fp, device)
    return _cached_plan(key, lambda: _capi.DevicePlan.create(n, batch, factors, elem_bytes, mode,
                                                             table if uses_table else None, device))


_MODES = {"fast": _capi.MODE_FAST, "exact": _capi.MODE_EXACT, "permute": _capi.MODE_PERMUTE}


def _validate(x: np.ndarray, plan: StagePlan, table: Optional[TwiddleTable], trace) -> None:
    # tiled_fft.hpp:325-333
    _require(x.shape[-1] == plan.n_total, "fft_tiled: signal length does not match the plan")
    _require(plan.pass_count() >= 1, "fft_tiled: empty plan")
    if table is not None:
        _require(table.resolution >= plan.n_total and table.resolution % plan.n_total == 0,
                 "fft_tiled: signal length must divide the table resolution")
    if trace is not None:
        _require(getattr(trace, "bank_count", plan.bank_count) == plan.bank_count,
                 "fft_tiled: plan was built for a different bank count")


def fft_tiled(x, plan: StagePlan, table: Optional[TwiddleTable] = None, trace=None, threads: int = 1,
              mode: str = "fast", device: int = 0, _sign: int = _capi.FORWARD) -> np.ndarray:
    """tiled_fft.hpp:321-407 on the GPU. ``x``: complex64/complex128 array of
    shape (..., n); leading dimensions are a batch of independent transforms.
    ``threads`` keeps its host meaning and does not change the result (the
    reference guarantees thread invariance, test_tiled_fft.cpp:236-253).
    ``mode``: "fast" (product path, within tolerance) or "exact" (bit-identical
    to the reference; executes ``plan.factors`` with the table's roots)."""
    x = np.asarray(x)
    _require(x.dtype in (np.complex64, np.complex128), "fft_tiled: signal must be complex64 or complex128")
    _validate(x, plan, table, trace)
    if table is not None:
        _require(table.values.dtype == x.dtype, "fft_tiled: table precision does not match the signal")
    m = _MODES[mode]
    x = np.ascontiguousarray(x)
    batch = int(np.prod(x.shape[:-1])) if x.ndim > 1 else 1
    dp = _device_plan(plan.n_total, batch, plan.factors, x.dtype.itemsize, m, table, device)
    out = np.empty_like(x)
    dp.exec_host(x.ctypes.data, out.ctypes.data, _sign)
    return out


def ifft_tiled(x, plan: StagePlan, table: Optional[TwiddleTable] = None, mode: str = "fast",
               device: int = 0) -> np.ndarray:
    """tiled_fft.hpp:410-423 (conj -> fft_tiled -> conj * 1/n), on the GPU."""
    return fft_tiled(x, plan, table, mode=mode, device=device, _sign=_capi.INVERSE)


# ---- the reference's remaining public ops ----------------------------------------------------------
def fft_levelwise(x, table: Optional[TwiddleTable] = None, trace=None, device: int = 0,
                  _sign: int = _capi.FORWARD) -> np.ndarray:
    """fft_baseline.hpp:66-116 — the paper's previous method on the GPU: a
    bit-reversal sweep then one launch per radix-2 level in global memory.
    Bit-identical to the reference's fft_levelwise."""
    x = np.ascontiguousarray(np.asarray(x))
    n = x.shape[-1]
    _require(is_power_of_two(n) and n >= 2, "fft_levelwise: signal length must be a power of two >= 2")
    if table is not None:
        _require(table.resolution >= n and table.resolution % n == 0,
                 "fft_levelwise: signal length must divide the table resolution")
    batch = int(np.prod(x.shape[:-1])) if x.ndim > 1 else 1
    dp = _device_plan(n, batch, None, x.dtype.itemsize, _capi.MODE_LEVELWISE, table, device)
    out = np.empty_like(x)
    dp.exec_host(x.ctypes.data, out.ctypes.data, _sign)
    return out


def ifft_levelwise(x, table: Optional[TwiddleTable] = None, device: int = 0) -> np.ndarray:
    """fft_baseline.hpp:120-132."""
    return fft_levelwise(x, table, device=device, _sign=_capi.INVERSE)


def exchange_transpose(data, stage: int, plan: StagePlan, trace=None, device: int = 0) -> np.ndarray:
    """tiled_fft.hpp:179-203: one sweep applying the pass's store permutation, on the GPU."""
    data = np.ascontiguousarray(np.asarray(data))
    _require(1 <= stage <= plan.pass_count(), "exchange_transpose: stage out of range")
    _require(data.shape[-1] == plan.n_total, "exchange_transpose: signal length does not match the plan")
    if plan.pass_count() == 1:
        return data.copy()
    out = np.empty_like(data)
    _capi.exchange(data.ctypes.data, out.ctypes.data, plan.n_total, plan.factors, stage, data.dtype.itemsize, device)
    return out


class FastBuffer:
    """tiled_fft.hpp:38-71 — a rows x cols tile with `stride` slots between rows."""

    def __init__(self, rows, cols, stride, capacity, row_offset=0, dtype=np.complex128):
        _require(rows >= 1 and cols >= 1, "FastBuffer: empty tile")
        _require(stride >= cols, "FastBuffer: stride narrower than a row")
        _require(rows * cols <= capacity, "FastBuffer: tile exceeds capacity")
        self._rows, self._cols, self._stride, self._capacity = rows, cols, stride, capacity
        self._row_offset = row_offset
        self.cells = np.zeros((rows, stride), dtype=dtype)

    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def stride(self):
        return self._stride

    def capacity(self):
        return self._capacity

    def row_offset(self):
        return self._row_offset

    def set_row_offset(self, v):
        self._row_offset = v

    def at(self, r, c):
        return self.cells[r, c]

    def set(self, r, c, v):
        self.cells[r, c] = v

    def tile(self) -> np.ndarray:
        return self.cells[:, :self._cols]


def make_stage_buffer(plan: StagePlan, stage: int, dtype=np.complex128) -> FastBuffer:  # tiled_fft.hpp:75-80
    g = plan.stage(stage)
    return FastBuffer(g.rows_per_tile, g.fft_len, g.padded_stride, plan.tile_capacity, dtype=dtype)


def stage_row_fft(buf: FastBuffer, length: int, table: TwiddleTable, device: int = 0) -> None:
    """tiled_fft.hpp:129-146: in-place transform of each row of the tile, on the
    GPU (exact tier: bit-identical to the reference's bit-reverse + dit_levels)."""
    _require(is_power_of_two(length), "stage_row_fft: length must be a power of two")
    _require(length <= buf.capacity(), "stage_row_fft: length exceeds tile capacity")
    _require(length == buf.cols(), "stage_row_fft: length must match the tile row width")
    _require(table.resolution >= length and table.resolution % length == 0,
             "stage_row_fft: length must divide the table resolution")
    rows = np.ascontiguousarray(buf.tile()).astype(table.values.dtype)
    if length == 1:
        return
    dp = _device_plan(length, buf.rows(), (length,), rows.dtype.itemsize, _capi.MODE_EXACT, table, device)
    out = np.empty_like(rows)
    dp.exec_host(rows.ctypes.data, out.ctypes.data, _capi.FORWARD)
    buf.cells[:, :length] = out


def apply_interstage_twiddles(buf: FastBuffer, stage: int, plan: StagePlan, table: TwiddleTable,
                              device: int = 0) -> None:
    """tiled_fft.hpp:153-172, on the GPU (bit-identical)."""
    _require(plan.pass_count() >= 1, "apply_interstage_twiddles: empty plan")
    _require(1 <= stage < plan.pass_count(), "apply_interstage_twiddles: stage must be an inter-pass boundary")
    g = plan.stage(stage)
    _require(buf.cols() == g.fft_len, "apply_interstage_twiddles: tile width does not match the pass")
    _require(buf.row_offset() + buf.rows() <= g.rows, "apply_interstage_twiddles: tile rows fall outside the pass grid")
    _require(table.resolution >= g.sub_len and table.resolution % g.sub_len == 0,
             "apply_interstage_twiddles: sub-transform length must divide the table resolution")
    t = np.ascontiguousarray(buf.tile()).astype(table.values.dtype)
    out = np.empty_like(t)
    _capi.interstage_scale(t.ctypes.data, out.ctypes.data, buf.rows(), buf.cols(), buf.row_offset(), g.rows_per_sub,
                           g.sub_len, table.values.ctypes.data, table.resolution, t.dtype.itemsize, device)
    buf.cells[:, :buf.cols()] = out


def fft2_tiled(x, device: int = 0, inverse: bool = False) -> np.ndarray:
    """2D transform of row-major (..., ny, nx) images: rows, then columns
    (the BASELINE.md recipe; the reference has no 2D entry point)."""
    x = np.ascontiguousarray(np.asarray(x))
    _require(x.ndim >= 2, "fft2_tiled: need (..., ny, nx)")
    ny, nx = x.shape[-2:]
    batch = int(np.prod(x.shape[:-2])) if x.ndim > 2 else 1
    key = ("2d", ny, nx, batch, x.dtype.itemsize, device)
    dp = _cached_plan(key, lambda: _capi.DevicePlan.create_2d(ny, nx, batch, x.dtype.itemsize, device))
    out = np.empty_like(x)
    dp.exec_host(x.ctypes.data, out.ctypes.data, _capi.INVERSE if inverse else _capi.FORWARD)
    return out


def fft_tiled_device(x, plan: StagePlan, out=None, mode: str = "fast", inverse: bool = False, device_plan=None):
    """Device-resident variant: ``x`` is a CUDA torch tensor (complex64 or
    complex128, shape (..., n)); runs on the tensor's current stream."""
    import torch
    _require(x.is_cuda and x.is_contiguous(), "fft_tiled_device: x must be a contiguous CUDA tensor")
    _require(x.shape[-1] == plan.n_total, "fft_tiled: signal length does not match the plan")
    if out is None:
        out = torch.empty_like(x)
    batch = x.numel() // plan.n_total
    dp = device_plan or _device_plan(plan.n_total, batch, plan.factors, x.element_size(), _MODES[mode], None,
                                     x.device.index)
    dp.exec_device(x.data_ptr(), out.data_ptr(), _capi.INVERSE if inverse else _capi.FORWARD,
                   torch.cuda.current_stream(x.device).cuda_stream)
    return out
