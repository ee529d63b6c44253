"""Multi-GPU execution.

* Batched / 2D transforms shard the batch (or the images) over ranks with no
  collective on the data path: ``shard_rows`` gives each rank its contiguous
  share and results are bit-identical to the single-GPU run (the GPU kernels do
  not depend on how many transforms a launch holds — the same thread-count
  invariance the reference guarantees, test_tiled_fft.cpp:236-253).

* A single 1D transform too large for one GPU runs as a four-step transform
  N = N1 x N2 over G ranks (``DistributedFFT``): the reference's own pass
  structure lifted to GPUs. Pass 1 (the comb pass, tiled_fft.hpp:252-294:
  column FFTs of length N1 plus the inter-pass root W_N^{r k1}) runs on the
  rank's column slab, and its store IS the exchange — spectrum row k1 belongs
  to rank k1 / (N1/G) (stage_plan.hpp:164-170). Two exchange transports:
    - ``"p2p"``: the pass-1 kernel writes its results straight into the other
      ranks' row slabs, mapped into this process with CUDA IPC, so the
      transpose rides NVLink inside the kernel, overlapped tile by tile with the
      butterflies (the fused compute + all-to-all);
    - ``"nccl"``: pass 1 writes per-destination staging blocks, then one
      ``all_to_all_single`` (NCCL grouped send/recv); pass 2 reads the receive
      buffer [src][k1][c] through a 5-D tensor map (one strided re-assembly
      copy only when the row plan is a single pass). The comparison path.
  With GPU ops the p2p step is ``tilefft_dist_exec``: pass 1, a one-thread
  peer-flag barrier kernel and pass 2 queued on one stream (no host
  synchronisation, CUDA-graph capturable).
  Pass 2 is the row FFT of length N2 on the rank's row slab (local multi-pass).

Layouts (rank g, C = N2/G, R = N1/G):
  input  column slab [N1][C]:  x[g*C + c + N2*n1]
  output row slab    [R][N2]:  X[(g*R + k1) + N1*k2]   (digit-interleaved slabs)
"""
from __future__ import annotations

import numpy as np

from . import _capi


def shard_rows(total: int, world: int, rank: int):
    """Contiguous [begin, end) share of `total` independent transforms."""
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def four_step_layout(n: int, world: int):
    """(N1, N2, C, R) of the distributed split (mirrors tilefft_dist_plan_create)."""
    n1 = min(1024, n >> 7)
    n2 = n // n1
    return n1, n2, n2 // world, n1 // world


def column_slab(x: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Rank `rank`'s input slab [N1][C] of a natural-order signal x."""
    n1, n2, c, _ = four_step_layout(x.shape[-1], world)
    return np.ascontiguousarray(x.reshape(n1, n2)[:, rank * c:(rank + 1) * c])


def natural_block(x: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Rank `rank`'s contiguous 1/world of a natural-order array (forward_natural's I/O layout)."""
    m = x.shape[-1] // world
    return np.ascontiguousarray(x[rank * m:(rank + 1) * m])


def assemble_output(slabs, n: int) -> np.ndarray:
    """Natural-order spectrum from every rank's row slab [R][N2]."""
    world = len(slabs)
    n1, n2, _, r = four_step_layout(n, world)
    rows = np.concatenate([np.asarray(s).reshape(r, n2) for s in slabs], axis=0)  # [k1][k2]
    return np.ascontiguousarray(rows.T).reshape(n)  # X[k1 + N1*k2]


class GpuOps:
    """The rank-local steps on the B200 through the C ABI."""

    def __init__(self, n, world, rank, device, elem_bytes=8):
        import torch
        self.torch = torch
        self.device = device
        self.plan = _capi.DistPlan.create_dist(n, world, rank, elem_bytes, device)
        lay = self.plan.layout()
        self.n1, self.n2, self.c, self.r = lay["n1"], lay["n2"], lay["cols_per_rank"], lay["rows_per_rank"]
        self.dtype = torch.complex64 if elem_bytes == 8 else torch.complex128

    def alloc(self, shape):
        return self.torch.empty(shape, dtype=self.dtype, device=f"cuda:{self.device}")

    @staticmethod
    def ptr(t):
        return t.data_ptr()

    def set_dests(self, ptrs, pitch, col_off):
        self.plan.set_peers(ptrs, pitch, col_off)

    def stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def pass1(self, slab, sign):
        self.plan.pass1(slab.data_ptr(), sign, self.stream())

    def pass2(self, rows, out, sign):
        self.plan.pass2(rows.data_ptr(), out.data_ptr(), sign, self.stream())

    def pass2_blocks(self, recv, out, sign):
        """pass 2 reading the all-to-all receive buffer [src][R][C] in place (raises if the row plan is one pass)."""
        self.plan.pass2_blocks(recv.data_ptr(), out.data_ptr(), sign, self.stream())

    def sync(self):
        self.torch.cuda.synchronize(self.device)

    def ipc_handle(self, t):
        return _capi.ipc_handle(t if isinstance(t, int) else t.data_ptr())

    def flag_buffer(self):
        return self.plan.flag_buffer()

    def set_flags(self, ptrs):
        self.plan.set_flags(ptrs)

    def step(self, slab, out, sign):
        """pass 1 (peer stores) -> device peer-flag barrier -> pass 2, no host synchronisation."""
        self.plan.exec_step(slab.data_ptr(), out.data_ptr(), sign, self.stream())

    def ipc_open(self, h):
        return _capi.ipc_open(h)


class DistributedFFT:
    """One length-n transform over the ranks of ``torch.distributed`` (or a
    single process when it is not initialised)."""

    def __init__(self, n: int, exchange: str = "p2p", ops=None, device: int = 0, elem_bytes: int = 8):
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.world = self.dist.get_world_size() if self.dist else 1
        self.rank = self.dist.get_rank() if self.dist else 0
        self.n = n
        self.exchange = exchange if self.world > 1 else "local"
        self.ops = ops or GpuOps(n, self.world, self.rank, device, elem_bytes)
        o = self.ops
        self.rows = o.alloc((o.r, o.n2))
        self._opened = []
        self._it = 0
        if self.exchange == "local":
            o.set_dests([o.ptr(self.rows)], o.n2, 0)
        elif self.exchange == "p2p":
            # Two row slabs used alternately: a fast rank's pass 1 of call i+1
            # writes the other slab, never the one a slower peer's pass 2 of
            # call i may still be reading (the barrier of call i orders call
            # i-1's pass 2 before every pass-1 store of call i+1).
            self._slabs = [self.rows, o.alloc((o.r, o.n2))]
            self._dests = []
            for slab in self._slabs:
                handles = [None] * self.world
                self.dist.all_gather_object(handles, o.ipc_handle(slab))
                ptrs = []
                for g, h in enumerate(handles):
                    if g == self.rank:
                        ptrs.append(o.ptr(slab))
                    else:
                        p = o.ipc_open(h)
                        self._opened.append(p)
                        ptrs.append(p)
                self._dests.append(ptrs)
            o.set_dests(self._dests[0], o.n2, self.rank * o.c)
            # device-side barrier words (GPU ops): every rank's flag buffer, own included
            self.device_barrier = hasattr(o, "flag_buffer")
            if self.device_barrier:
                mine = o.flag_buffer()
                handles = [None] * self.world
                self.dist.all_gather_object(handles, o.ipc_handle(mine))
                flags = []
                for g, h in enumerate(handles):
                    if g == self.rank:
                        flags.append(mine)
                    else:
                        p = o.ipc_open(h)
                        self._opened.append(p)
                        flags.append(p)
                o.set_flags(flags)
        elif self.exchange == "nccl":
            self.stage = o.alloc((self.world, o.r, o.c))
            self.recv = o.alloc((self.world, o.r, o.c))
            o.set_dests([o.ptr(self.stage[d]) for d in range(self.world)], o.c, 0)
        else:
            raise ValueError(f"unknown exchange {exchange!r}")

    def forward(self, col_slab, out=None, inverse: bool = False):
        """col_slab: this rank's [N1][C] slab; returns its [R][N2] output slab."""
        o = self.ops
        sign = _capi.INVERSE if inverse else _capi.FORWARD
        if out is None:
            out = o.alloc((o.r, o.n2))
        if self.exchange == "p2p":
            b = self._it & 1
            self._it += 1
            self.rows = self._slabs[b]
            o.set_dests(self._dests[b], o.n2, self.rank * o.c)
            if self.device_barrier:
                o.step(col_slab, out, sign)  # stream-ordered: no host sync, graph-capturable per slab parity
                return out
        o.pass1(col_slab, sign)
        if self.exchange == "p2p":
            o.sync()              # this rank's peer stores are complete ...
            self.dist.barrier()   # ... and so are everyone else's into our slab
        elif self.exchange == "nccl":
            self.dist.all_to_all_single(self.recv, self.stage)
            if getattr(self, "_blocks", hasattr(o, "pass2_blocks")):
                try:  # pass 2 reads the [src][k1][c] receive buffer through a 5-D tensor map: no re-assembly
                    o.pass2_blocks(self.recv, out, sign)
                    self._blocks = True
                    return out
                except ValueError:
                    self._blocks = False  # single-pass row plan: assemble the rows instead
            # [src][k1][c] -> [k1][src*C + c]: one strided copy
            self.rows.view(o.r, self.world, o.c).copy_(self.recv.permute(1, 0, 2))
        o.pass2(self.rows, out, sign)
        return out

    def forward_natural(self, x_block, inverse: bool = False):
        """Natural-order block I/O (SURVEY §8e option): x_block is this rank's contiguous 1/G of the signal,
        x[g·N/G : (g+1)·N/G]; returns this rank's contiguous 1/G of the spectrum, X[g·N/G : (g+1)·N/G].

        Costs one all-to-all before the four-step exchange (rows n1 ∈ [gR, (g+1)R) of the [N1][N2] signal
        matrix -> the column slab) and one after it (the digit-interleaved row slab -> natural blocks), each
        an ``all_to_all_single`` plus one strided copy; the in-kernel exchange of pass 1 is unchanged."""
        o = self.ops
        G, R, C, N1, N2 = self.world, o.r, o.c, o.n1, o.n2
        M = N2 // G
        if G == 1:
            return self.forward(x_block.reshape(N1, N2), inverse=inverse).reshape(-1)
        # 1. block rows [R][N2] -> per-destination column blocks [G][R][C] -> column slab [N1][C]
        send = x_block.reshape(R, G, C).permute(1, 0, 2).contiguous()
        col = o.alloc((G, R, C))
        self.dist.all_to_all_single(col, send)
        y = self.forward(col.reshape(N1, C), inverse=inverse)  # row slab [R][N2]: X[(gR + k1) + N1 k2]
        # 2. rows k1 of this rank, spectrum columns k2 of each destination's natural block -> [G][R][M]
        send2 = y.reshape(R, G, M).permute(1, 0, 2).contiguous()
        recv2 = o.alloc((G, R, M))
        self.dist.all_to_all_single(recv2, send2)
        # recv2[s][k1 - sR][m] = X[k1 + N1 (gM + m)]: natural order is m-major, k1-minor
        return recv2.reshape(N1, M).t().contiguous().reshape(-1)

    def close(self):
        for p in self._opened:
            try:
                _capi.ipc_close(p)
            except Exception:
                pass
        self._opened = []
