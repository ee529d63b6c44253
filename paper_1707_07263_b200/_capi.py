"""ctypes binding of the C ABI in include/tilefft_b200.h.

Loads the in-tree ``libtilefft_b200.so`` (built by ``__graft_entry__.build()`` /
``make -C paper_1707_07263_b200/csrc``). There is deliberately no fallback: if
the library is missing, or no sm_100 device is present when a plan is created,
the call raises — the product path never runs on the CPU.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtilefft_b200.so")

OK = 0
EINVAL = 22
ENODEV = 19
ENOMEM = 12
ECUDA = 1001
ENCCL = 1002

MODE_FAST = 0
MODE_EXACT = 1
MODE_PERMUTE = 2
MODE_LEVELWISE = 3
FORWARD = -1
INVERSE = +1


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("batch", ctypes.c_uint64),
        ("ny", ctypes.c_uint64),
        ("nx", ctypes.c_uint64),
        ("elem_bytes", ctypes.c_uint32),
        ("mode", ctypes.c_uint32),
        ("is_2d", ctypes.c_uint32),
        ("passes", ctypes.c_uint32),
        ("factors", ctypes.c_uint64 * 16),
        ("launches_per_exec", ctypes.c_uint32),
        ("workspace_bytes", ctypes.c_uint64),
        ("table_bytes", ctypes.c_uint64),
    ]


# Every symbol include/tilefft_b200.h declares (tests check the exports).
EXPORTS = (
    "tilefft_plan_create",
    "tilefft_plan_create_2d",
    "tilefft_exec_c2c",
    "tilefft_exec_c2c_host",
    "tilefft_exec_c2c_timed",
    "tilefft_plan_destroy",
    "tilefft_plan_info",
    "tilefft_build_twiddle",
    "tilefft_account",
    "tilefft_exchange",
    "tilefft_interstage_scale",
    "tilefft_dist_plan_create",
    "tilefft_dist_layout",
    "tilefft_dist_set_peers",
    "tilefft_dist_exec_pass1",
    "tilefft_dist_exec_pass2",
    "tilefft_dist_exec_pass2_blocks",
    "tilefft_dist_flag_buffer",
    "tilefft_dist_set_flags",
    "tilefft_dist_exec",
    "tilefft_ipc_get_handle",
    "tilefft_ipc_open_handle",
    "tilefft_ipc_close_handle",
    "tilefft_last_error",
    "tilefft_version",
)

_lib = None
_lock = threading.Lock()


class TilefftError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        u64, u32, i32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p
        lib.tilefft_plan_create.argtypes = [ctypes.POINTER(vp), u64, u64, ctypes.POINTER(u64), u32, u32, u32, vp,
                                            u64, i32]
        lib.tilefft_plan_create_2d.argtypes = [ctypes.POINTER(vp), u64, u64, u64, u32, i32]
        lib.tilefft_exec_c2c.argtypes = [vp, vp, vp, i32, vp]
        lib.tilefft_exec_c2c_host.argtypes = [vp, vp, vp, i32]
        lib.tilefft_exec_c2c_timed.argtypes = [vp, vp, vp, i32, vp, i32, ctypes.POINTER(ctypes.c_float), i32]
        lib.tilefft_plan_destroy.argtypes = [vp]
        lib.tilefft_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        lib.tilefft_build_twiddle.argtypes = [u64, u32, vp]
        lib.tilefft_account.argtypes = [u64, u64, u32, ctypes.POINTER(u64)]
        lib.tilefft_exchange.argtypes = [vp, vp, u64, ctypes.POINTER(u64), u32, u32, u32, i32]
        lib.tilefft_interstage_scale.argtypes = [vp, vp, u64, u64, u64, u64, u64, vp, u64, u32, i32]
        lib.tilefft_dist_plan_create.argtypes = [ctypes.POINTER(vp), u64, u32, u32, u32, i32]
        lib.tilefft_dist_layout.argtypes = [vp] + [ctypes.POINTER(u64)] * 4
        lib.tilefft_dist_set_peers.argtypes = [vp, ctypes.POINTER(vp), u32, u64, u64]
        lib.tilefft_dist_exec_pass1.argtypes = [vp, vp, i32, vp]
        lib.tilefft_dist_exec_pass2.argtypes = [vp, vp, vp, i32, vp]
        lib.tilefft_ipc_get_handle.argtypes = [vp, vp, ctypes.POINTER(u64)]
        lib.tilefft_dist_exec_pass2_blocks.argtypes = [vp, vp, vp, i32, vp]
        lib.tilefft_dist_flag_buffer.argtypes = [vp, ctypes.POINTER(vp)]
        lib.tilefft_dist_set_flags.argtypes = [vp, ctypes.POINTER(vp), u32]
        lib.tilefft_dist_exec.argtypes = [vp, vp, vp, i32, vp]
        lib.tilefft_ipc_open_handle.argtypes = [vp, u64, ctypes.POINTER(vp)]
        lib.tilefft_ipc_close_handle.argtypes = [vp]
        lib.tilefft_last_error.restype = ctypes.c_char_p
        lib.tilefft_debug_two_watchdog.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), i32]  # diagnostics only
        lib.tilefft_version.restype = ctypes.c_char_p
        for name in ("tilefft_plan_create", "tilefft_plan_create_2d", "tilefft_exec_c2c", "tilefft_exec_c2c_host",
                     "tilefft_plan_destroy", "tilefft_plan_info", "tilefft_build_twiddle", "tilefft_account",
                     "tilefft_exchange",
                     "tilefft_interstage_scale", "tilefft_dist_plan_create", "tilefft_dist_layout",
                     "tilefft_dist_set_peers", "tilefft_dist_exec_pass1", "tilefft_dist_exec_pass2",
                     "tilefft_dist_exec_pass2_blocks",
                     "tilefft_dist_flag_buffer", "tilefft_dist_set_flags", "tilefft_dist_exec",
                     "tilefft_ipc_get_handle", "tilefft_ipc_open_handle", "tilefft_ipc_close_handle"):
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != OK:
        msg = load().tilefft_last_error().decode()
        if rc == EINVAL:
            # the reference throws std::invalid_argument (common.hpp:47-51)
            raise ValueError(msg)
        raise TilefftError(rc, msg)


class DevicePlan:
    """Owning wrapper of a ``tilefft_plan_t``."""

    def __init__(self, handle: int, lib: ctypes.CDLL):
        self._h = ctypes.c_void_p(handle)
        self._lib = lib

    @classmethod
    def create(cls, n, batch=1, factors=None, elem_bytes=8, mode=MODE_FAST, table=None, device=0):
        lib = load()
        h = ctypes.c_void_p()
        fac = None
        nf = 0
        if factors:
            nf = len(factors)
            fac = (ctypes.c_uint64 * nf)(*[int(f) for f in factors])
        tv, tres = None, 0
        if table is not None:
            tv = ctypes.c_void_p(table.values.ctypes.data)
            tres = int(table.resolution)
        check(lib.tilefft_plan_create(ctypes.byref(h), int(n), int(batch), fac, nf, int(elem_bytes), int(mode), tv,
                                      tres, int(device)))
        return cls(h.value, lib)

    @classmethod
    def create_2d(cls, ny, nx, batch=1, elem_bytes=8, device=0):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.tilefft_plan_create_2d(ctypes.byref(h), int(ny), int(nx), int(batch), int(elem_bytes), int(device)))
        return cls(h.value, lib)

    def exec_device(self, d_in: int, d_out: int, sign: int = FORWARD, stream: int = 0) -> None:
        check(self._lib.tilefft_exec_c2c(self._h, ctypes.c_void_p(d_in), ctypes.c_void_p(d_out), int(sign),
                                         ctypes.c_void_p(stream)))

    def exec_host(self, h_in: int, h_out: int, sign: int = FORWARD) -> None:
        check(self._lib.tilefft_exec_c2c_host(self._h, ctypes.c_void_p(h_in), ctypes.c_void_p(h_out), int(sign)))

    def exec_timed(self, d_in: int, d_out: int, sign: int = FORWARD, stream: int = 0, reps: int = 10) -> list:
        """Per-pass mean CUDA-event durations (ms) over `reps` direct executions (measurement only)."""
        n = int(self.info()["passes"])
        ms = (ctypes.c_float * max(1, n))()
        check(self._lib.tilefft_exec_c2c_timed(self._h, ctypes.c_void_p(d_in), ctypes.c_void_p(d_out), int(sign),
                                               ctypes.c_void_p(stream), int(reps), ms, n))
        return [float(ms[i]) for i in range(n)]

    def info(self) -> dict:
        pi = PlanInfo()
        check(self._lib.tilefft_plan_info(self._h, ctypes.byref(pi)))
        d = {k: getattr(pi, k) for k, _ in PlanInfo._fields_ if k != "factors"}
        d["factors"] = [int(pi.factors[i]) for i in range(min(pi.passes, 16))]
        return d

    def close(self) -> None:
        if self._h and self._h.value:
            self._lib.tilefft_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exchange(h_in: int, h_out: int, n: int, factors, stage: int, elem_bytes: int, device: int = 0) -> None:
    fac = (ctypes.c_uint64 * len(factors))(*[int(f) for f in factors])
    check(load().tilefft_exchange(ctypes.c_void_p(h_in), ctypes.c_void_p(h_out), int(n), fac, len(factors),
                                  int(stage), int(elem_bytes), int(device)))


def interstage_scale(h_in: int, h_out: int, rows: int, cols: int, row0: int, rows_per_sub: int, sub_len: int,
                     table_ptr: int, resolution: int, elem_bytes: int, device: int = 0) -> None:
    check(load().tilefft_interstage_scale(ctypes.c_void_p(h_in), ctypes.c_void_p(h_out), int(rows), int(cols),
                                          int(row0), int(rows_per_sub), int(sub_len), ctypes.c_void_p(table_ptr),
                                          int(resolution), int(elem_bytes), int(device)))


ACCOUNT_TILED = 0
ACCOUNT_LEVELWISE = 1
ACCESS_STATS_FIELDS = ("slow_elem_reads", "slow_elem_writes", "slow_transactions", "fast_accesses",
                       "bank_conflict_cycles", "barriers", "twiddle_fetches")


def account(n: int, tile_capacity: int, algorithm: int) -> dict:
    """The reference's cost model (memsim.hpp) through tilefft_account: host only."""
    out = (ctypes.c_uint64 * 7)()
    check(load().tilefft_account(int(n), int(tile_capacity), int(algorithm), out))
    return dict(zip(ACCESS_STATS_FIELDS, (int(v) for v in out)))


def build_twiddle(resolution: int, elem_bytes: int, out_ptr: int) -> None:
    check(load().tilefft_build_twiddle(int(resolution), int(elem_bytes), ctypes.c_void_p(out_ptr)))


class DistPlan(DevicePlan):
    """One rank's share of a distributed four-step transform (tilefft_dist_*)."""

    @classmethod
    def create_dist(cls, n, nranks, rank, elem_bytes=8, device=0):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.tilefft_dist_plan_create(ctypes.byref(h), int(n), int(nranks), int(rank), int(elem_bytes),
                                           int(device)))
        return cls(h.value, lib)

    def layout(self):
        v = [ctypes.c_uint64() for _ in range(4)]
        check(self._lib.tilefft_dist_layout(self._h, *[ctypes.byref(x) for x in v]))
        return dict(n1=v[0].value, n2=v[1].value, cols_per_rank=v[2].value, rows_per_rank=v[3].value)

    def set_peers(self, ptrs, row_pitch, col_off):
        arr = (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
        check(self._lib.tilefft_dist_set_peers(self._h, arr, len(ptrs), int(row_pitch), int(col_off)))

    def pass1(self, d_slab, sign=FORWARD, stream=0):
        check(self._lib.tilefft_dist_exec_pass1(self._h, ctypes.c_void_p(d_slab), int(sign), ctypes.c_void_p(stream)))

    def pass2(self, d_rows, d_out, sign=FORWARD, stream=0):
        check(self._lib.tilefft_dist_exec_pass2(self._h, ctypes.c_void_p(d_rows), ctypes.c_void_p(d_out), int(sign),
                                                ctypes.c_void_p(stream)))

    def pass2_blocks(self, d_recv, d_out, sign=FORWARD, stream=0):
        """pass 2 reading the all-to-all receive buffer [src][rows][cols] directly (tilefft_dist_exec_pass2_blocks)."""
        check(self._lib.tilefft_dist_exec_pass2_blocks(self._h, ctypes.c_void_p(d_recv), ctypes.c_void_p(d_out),
                                                       int(sign), ctypes.c_void_p(stream)))

    def flag_buffer(self) -> int:
        p = ctypes.c_void_p()
        check(self._lib.tilefft_dist_flag_buffer(self._h, ctypes.byref(p)))
        return p.value

    def set_flags(self, ptrs):
        arr = (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
        check(self._lib.tilefft_dist_set_flags(self._h, arr, len(ptrs)))

    def exec_step(self, d_slab, d_out, sign=FORWARD, stream=0):
        """pass 1 -> device barrier -> pass 2, stream-ordered (tilefft_dist_exec)."""
        check(self._lib.tilefft_dist_exec(self._h, ctypes.c_void_p(d_slab), ctypes.c_void_p(d_out), int(sign),
                                          ctypes.c_void_p(stream)))


def ipc_handle(dptr: int):
    """(64-byte CUDA IPC handle of the allocation holding dptr, byte offset of dptr inside it)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    check(load().tilefft_ipc_get_handle(ctypes.c_void_p(dptr), buf, ctypes.byref(off)))
    return buf.raw, off.value


def ipc_open(handle) -> int:
    raw, off = handle
    p = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(raw), 64)
    check(load().tilefft_ipc_open_handle(buf, int(off), ctypes.byref(p)))
    return p.value


def ipc_close(dptr: int) -> None:
    check(load().tilefft_ipc_close_handle(ctypes.c_void_p(dptr)))
