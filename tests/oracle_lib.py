"""ctypes access to the oracle — TEST INFRASTRUCTURE ONLY.

* ``Oracle``: the plain-C restatement (oracle/liboracle.so).
* ``Reference``: the reference's own headers compiled into
  oracle/_ref/libtilefft_ref.so (present when /root/reference was available at
  build time; the prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libtilefft_ref.so")

MAXP = 64


class OrcGeom(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("fft_len", "levels", "rows", "sub_len", "rows_per_sub",
                                                "padded_stride", "rows_per_tile", "tile_count")]


class OrcPlan(ctypes.Structure):
    _fields_ = [("n_total", ctypes.c_uint64), ("tile_capacity", ctypes.c_uint64), ("bank_count", ctypes.c_uint32),
                ("passes", ctypes.c_uint32), ("factors", ctypes.c_uint64 * MAXP), ("stages", OrcGeom * MAXP),
                ("sub_weights", ctypes.c_uint64 * MAXP), ("out_weights", ctypes.c_uint64 * MAXP)]


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _ensure_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, os.path.join(ORACLE_DIR, "liboracle.so")], check=True)


class Oracle:
    def __init__(self):
        _ensure_built()
        self.lib = ctypes.CDLL(ORACLE_SO)
        L = self.lib
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        L.orc_make_plan.argtypes = [u64, u64, u32, ctypes.POINTER(OrcPlan)]
        for suf in ("f32", "f64"):
            getattr(L, f"orc_build_twiddle_{suf}").argtypes = [u64, vp]
            getattr(L, f"orc_fft_tiled_{suf}").argtypes = [vp, vp, ctypes.POINTER(OrcPlan), vp, u64]
            getattr(L, f"orc_ifft_tiled_{suf}").argtypes = [vp, vp, ctypes.POINTER(OrcPlan), vp, u64]
            getattr(L, f"orc_fft_levelwise_{suf}").argtypes = [vp, vp, u64, vp, u64]
        L.orc_permute_tiled_f32.argtypes = [vp, vp, ctypes.POINTER(OrcPlan)]
        L.orc_dft_reference_f64.argtypes = [vp, vp, u64, ctypes.c_int, ctypes.c_int]
        L.orc_random_bench_signal.argtypes = [u64, u64, vp]
        L.orc_random_signal.argtypes = [u64, u64, vp]
        L.orc_splitmix_signal_f32.argtypes = [u64, u64, vp]
        L.orc_dft_bins_f32in.argtypes = [vp, u64, vp, u32, ctypes.c_int, u32, vp]
        L.orc_bit_reverse.argtypes = [u64, u32]
        L.orc_bit_reverse.restype = u64
        L.orc_gather_source_index.argtypes = [ctypes.POINTER(OrcPlan), u32, u64, u64]
        L.orc_gather_source_index.restype = u64
        L.orc_final_output_index.argtypes = [ctypes.POINTER(OrcPlan), u64, u64]
        L.orc_final_output_index.restype = u64
        L.orc_exchange_index_map.argtypes = [ctypes.POINTER(OrcPlan), u32, u64]
        L.orc_exchange_index_map.restype = u64

    # -- plan / table
    def make_plan(self, n, cap=1024, bank_count=16) -> OrcPlan:
        p = OrcPlan()
        rc = self.lib.orc_make_plan(n, cap, bank_count, ctypes.byref(p))
        if rc != 0:
            raise ValueError("make_plan: invalid argument")
        return p

    @staticmethod
    def factors(p: OrcPlan):
        return [int(p.factors[i]) for i in range(p.passes)]

    def twiddle(self, res, dtype=np.complex64) -> np.ndarray:
        t = np.empty(res, dtype=dtype)
        fn = self.lib.orc_build_twiddle_f32 if t.dtype == np.complex64 else self.lib.orc_build_twiddle_f64
        if fn(res, _ptr(t)) != 0:
            raise ValueError("build_twiddle_table: resolution must be a power of two >= 2")
        return t

    # -- transforms (single transform, or a batch along axis 0 when x is 2-D)
    def fft_tiled(self, x: np.ndarray, cap=1024, res=None, factors_plan=None, inverse=False) -> np.ndarray:
        x = np.ascontiguousarray(x)
        n = x.shape[-1]
        plan = factors_plan or self.make_plan(n, cap)
        res = res or n
        tbl = self.twiddle(res, x.dtype)
        suf = "f32" if x.dtype == np.complex64 else "f64"
        fn = getattr(self.lib, f"orc_{'ifft' if inverse else 'fft'}_tiled_{suf}")
        out = np.empty_like(x)
        for xi, oi in zip(x.reshape(-1, n), out.reshape(-1, n)):
            if fn(_ptr(xi), _ptr(oi), ctypes.byref(plan), _ptr(tbl), res) != 0:
                raise ValueError("fft_tiled: invalid argument")
        return out

    def permute_tiled(self, x: np.ndarray, cap=1024) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.complex64)
        out = np.empty_like(x)
        plan = self.make_plan(x.shape[-1], cap)
        self.lib.orc_permute_tiled_f32(_ptr(x), _ptr(out), ctypes.byref(plan))
        return out

    def fft_levelwise(self, x: np.ndarray, res=None) -> np.ndarray:
        x = np.ascontiguousarray(x)
        n = x.shape[-1]
        res = res or n
        tbl = self.twiddle(res, x.dtype)
        suf = "f32" if x.dtype == np.complex64 else "f64"
        out = np.empty_like(x)
        if getattr(self.lib, f"orc_fft_levelwise_{suf}")(_ptr(x), _ptr(out), n, _ptr(tbl), res) != 0:
            raise ValueError("fft_levelwise: invalid argument")
        return out

    def dft(self, x: np.ndarray, inverse=False) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.complex128)
        out = np.empty_like(x)
        self.lib.orc_dft_reference_f64(_ptr(x), _ptr(out), x.shape[-1], 1 if inverse else -1, 1 if inverse else 0)
        return out

    def fft2(self, img: np.ndarray, cap=1024) -> np.ndarray:
        """Rows then columns through fft_tiled (BASELINE.md §2 recipe)."""
        ny, nx = img.shape[-2:]
        rows = self.fft_tiled(img.reshape(-1, nx), cap).reshape(img.shape)
        cols = np.ascontiguousarray(np.swapaxes(rows, -1, -2))
        out = self.fft_tiled(cols.reshape(-1, ny), cap).reshape(cols.shape)
        return np.ascontiguousarray(np.swapaxes(out, -1, -2))

    # -- inputs
    def random_bench_signal(self, n, seed=1) -> np.ndarray:
        out = np.empty(n, dtype=np.complex128)
        self.lib.orc_random_bench_signal(n, seed, _ptr(out))
        return out

    def random_signal(self, n, seed) -> np.ndarray:
        out = np.empty(n, dtype=np.complex128)
        self.lib.orc_random_signal(n, seed, _ptr(out))
        return out

    def splitmix_signal(self, n, seed=1) -> np.ndarray:
        out = np.empty(n, dtype=np.complex64)
        self.lib.orc_splitmix_signal_f32(n, seed, _ptr(out))
        return out

    def dft_bins(self, x: np.ndarray, bins, inverse=False, threads=None) -> np.ndarray:
        """Exact fp64 DFT bins X[k] of a complex64 signal (O(N) per bin, threaded)."""
        x = np.ascontiguousarray(x, dtype=np.complex64)
        b = np.ascontiguousarray(np.asarray(bins, dtype=np.uint64))
        out = np.empty(len(b), dtype=np.complex128)
        rc = self.lib.orc_dft_bins_f32in(_ptr(x), x.shape[-1], _ptr(b), len(b), 1 if inverse else -1,
                                         int(threads or os.cpu_count() or 1), _ptr(out))
        if rc != 0:
            raise ValueError("dft_bins: invalid argument")
        return out


class Reference:
    """The reference itself (compiled headers). Raises if not built."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = ctypes.CDLL(REF_SO)
        L = self.lib
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        for suf in ("f32", "f64"):
            getattr(L, f"ref_fft_tiled_{suf}").argtypes = [vp, vp, u64, u64, u64, u32]
            getattr(L, f"ref_ifft_tiled_{suf}").argtypes = [vp, vp, u64, u64, u64]
            getattr(L, f"ref_fft_levelwise_{suf}").argtypes = [vp, vp, u64, u64]
            getattr(L, f"ref_dft_reference_{suf}").argtypes = [vp, vp, u64]
            getattr(L, f"ref_build_twiddle_{suf}").argtypes = [u64, vp]
        L.ref_make_plan.argtypes = [u64, u64, ctypes.POINTER(u32), vp, vp, vp, vp]
        L.ref_random_bench_signal.argtypes = [u64, u64, vp]
        L.ref_exchange_index_map.argtypes = [u64, u64, u32, u64]
        L.ref_exchange_index_map.restype = u64
        L.ref_gather_source_index.argtypes = [u64, u64, u32, u64, u64]
        L.ref_gather_source_index.restype = u64
        L.ref_exchange_transpose_f64.argtypes = [vp, vp, u64, u64, u32]
        L.ref_ctx_create.argtypes = [u64, u64]
        L.ref_ctx_create.restype = vp
        L.ref_ctx_destroy.argtypes = [vp]
        L.ref_ctx_exec_single.argtypes = [vp, vp, vp, u32]
        L.ref_ctx_exec_batched.argtypes = [vp, vp, vp, u64, u32]
        L.ref_hardware_concurrency.restype = u32
        L.ref_account_tiled.argtypes = [u64, u64, vp]
        L.ref_account_levelwise.argtypes = [u64, vp]

    def fft_tiled(self, x, cap=1024, res=None, threads=1, inverse=False):
        x = np.ascontiguousarray(x)
        n = x.shape[-1]
        res = res or n
        suf = "f32" if x.dtype == np.complex64 else "f64"
        out = np.empty_like(x)
        for xi, oi in zip(x.reshape(-1, n), out.reshape(-1, n)):
            if inverse:
                rc = getattr(self.lib, f"ref_ifft_tiled_{suf}")(_ptr(xi), _ptr(oi), n, cap, res)
            else:
                rc = getattr(self.lib, f"ref_fft_tiled_{suf}")(_ptr(xi), _ptr(oi), n, cap, res, threads)
            if rc != 0:
                raise ValueError("fft_tiled: invalid argument")
        return out

    def fft_tiled_batched(self, x, cap=1024, threads=None):
        """fp32 rows of x (shape (batch, n)) through the reference's fft_tiled,
        `threads` std::threads each calling fft_tiled(threads=1)."""
        x = np.ascontiguousarray(x, dtype=np.complex64)
        n = x.shape[-1]
        batch = x.size // n
        out = np.empty_like(x)
        ctx = self.lib.ref_ctx_create(n, cap)
        if not ctx:
            raise ValueError("fft_tiled: invalid argument")
        try:
            self.lib.ref_ctx_exec_batched(ctx, _ptr(x), _ptr(out), batch, int(threads or os.cpu_count() or 1))
        finally:
            self.lib.ref_ctx_destroy(ctx)
        return out

    def fft2(self, img, cap=1024, threads=None):
        """fp32 2D transform as rows then columns through fft_tiled (BASELINE.md §2 recipe;
        the reference has no 2D entry point)."""
        ny, nx = img.shape[-2:]
        rows = self.fft_tiled_batched(img.reshape(-1, nx), cap, threads).reshape(img.shape)
        cols = np.ascontiguousarray(np.swapaxes(rows, -1, -2))
        del rows
        out = self.fft_tiled_batched(cols.reshape(-1, ny), cap, threads).reshape(cols.shape)
        return np.ascontiguousarray(np.swapaxes(out, -1, -2))

    def account_tiled(self, n, cap=1024):
        """memsim.hpp account_tiled(make_plan(n, cap)): 7 counters in AccessStats order."""
        out = np.zeros(7, np.uint64)
        if self.lib.ref_account_tiled(n, cap, _ptr(out)) != 0:
            raise ValueError("account_tiled: invalid argument")
        return [int(v) for v in out]

    def account_levelwise(self, n):
        out = np.zeros(7, np.uint64)
        if self.lib.ref_account_levelwise(n, _ptr(out)) != 0:
            raise ValueError("account_levelwise: invalid argument")
        return [int(v) for v in out]

    def fft_levelwise(self, x, res=None):
        x = np.ascontiguousarray(x)
        suf = "f32" if x.dtype == np.complex64 else "f64"
        out = np.empty_like(x)
        if getattr(self.lib, f"ref_fft_levelwise_{suf}")(_ptr(x), _ptr(out), x.shape[-1], res or x.shape[-1]) != 0:
            raise ValueError("fft_levelwise: invalid argument")
        return out

    def dft(self, x):
        x = np.ascontiguousarray(x)
        suf = "f32" if x.dtype == np.complex64 else "f64"
        out = np.empty_like(x)
        getattr(self.lib, f"ref_dft_reference_{suf}")(_ptr(x), _ptr(out), x.shape[-1])
        return out

    def twiddle(self, res, dtype=np.complex64):
        t = np.empty(res, dtype=dtype)
        suf = "f32" if t.dtype == np.complex64 else "f64"
        if getattr(self.lib, f"ref_build_twiddle_{suf}")(res, _ptr(t)) != 0:
            raise ValueError("build_twiddle_table: invalid")
        return t

    def make_plan(self, n, cap=1024):
        passes = ctypes.c_uint32()
        fac = np.zeros(MAXP, np.uint64)
        geom = np.zeros(8 * MAXP, np.uint64)
        sw = np.zeros(MAXP, np.uint64)
        ow = np.zeros(MAXP, np.uint64)
        if self.lib.ref_make_plan(n, cap, ctypes.byref(passes), _ptr(fac), _ptr(geom), _ptr(sw), _ptr(ow)) != 0:
            raise ValueError("make_plan: invalid argument")
        p = passes.value
        return dict(factors=[int(v) for v in fac[:p]], geom=geom[:8 * p].reshape(p, 8).astype(int).tolist(),
                    sub_weights=[int(v) for v in sw[:max(p - 1, 0)]], out_weights=[int(v) for v in ow[:p]])

    def random_bench_signal(self, n, seed=1):
        out = np.empty(n, dtype=np.complex128)
        self.lib.ref_random_bench_signal(n, seed, _ptr(out))
        return out

    def exchange_transpose(self, x, cap, stage):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        out = np.empty_like(x)
        if self.lib.ref_exchange_transpose_f64(_ptr(x), _ptr(out), x.shape[-1], cap, stage) != 0:
            raise ValueError("exchange_transpose: invalid")
        return out


def available_reference() -> bool:
    return os.path.exists(REF_SO)


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    assert a.shape == b.shape, (a.shape, b.shape)
    num = den = 0.0
    step = 1 << 24  # chunked: 2^30-point arrays would need 32 GB of complex128 temporaries
    for s in range(0, a.size, step):
        ac = a[s:s + step].astype(np.complex128)
        bc = b[s:s + step].astype(np.complex128)
        d = ac - bc
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(bc, bc).real)
    return float(np.sqrt(num) / (np.sqrt(den) if den > 0 else 1.0))
