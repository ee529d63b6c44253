"""Multi-GPU paths.

CPU (gloo, world size 2): the distributed four-step orchestration — column
slabs in, pass-1 scatter into per-destination blocks, all_to_all_single,
re-assembly, pass 2 — with the rank-local steps done by the oracle (test
infrastructure standing in for the GPU kernels), checked against the oracle's
single-process fft_tiled; plus batch sharding.
GPU (one device): the fused pass-1 kernel scattering into G row slabs
("virtual ranks" on one B200; on a multi-GPU box the same kernel writes
through CUDA-IPC-mapped peer pointers), checked against the oracle.
"""
import math
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    """Rank-local steps on the CPU through the oracle (tests only)."""

    def __init__(self, n, world, rank):
        sys.path.insert(0, HERE)
        from oracle_lib import Oracle
        from paper_1707_07263_b200.distributed import four_step_layout
        self.O = Oracle()
        self.n, self.world, self.rank = n, world, rank
        self.n1, self.n2, self.c, self.r = four_step_layout(n, world)

    def alloc(self, shape):
        import torch
        return torch.zeros(shape, dtype=torch.complex128)

    @staticmethod
    def ptr(t):
        return t

    def set_dests(self, dests, pitch, col_off):
        self.dests, self.pitch, self.col_off = [d.reshape(-1) for d in dests], pitch, col_off

    def pass1(self, slab, sign):
        x = slab.numpy() if hasattr(slab, "numpy") else slab
        cols = self.O.fft_tiled(np.ascontiguousarray(x.T))  # [C][N1], FFT over n1
        r = self.rank * self.c + np.arange(self.c)[:, None]
        k = np.arange(self.n1)[None, :]
        w = np.exp(-2j * np.pi * ((r * k) % self.n) / self.n)
        y = cols * w  # [C][N1]
        for kk in range(self.n1):
            d, kr = divmod(kk, self.r)
            dst = self.dests[d]
            base = kr * self.pitch + self.col_off
            dst[base:base + self.c] = __import__("torch").from_numpy(np.ascontiguousarray(y[:, kk]))

    def pass2(self, rows, out, sign):
        out.copy_(__import__("torch").from_numpy(self.O.fft_tiled(rows.numpy())))

    def sync(self):
        pass


class SharedMemOracleOps(OracleOps):
    """OracleOps whose row slabs live in shared-memory files, so the "p2p"
    exchange (pass 1 storing straight into the peers' slabs, CUDA IPC on the
    GPU) runs across processes on the CPU: ipc_handle = the file name."""

    _count = 0

    def alloc(self, shape):
        import tempfile
        import torch
        SharedMemOracleOps._count += 1
        fd, path = tempfile.mkstemp(prefix=f"tilefft_r{self.rank}_", dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
        os.close(fd)
        nbytes = int(np.prod(shape)) * 16
        t = torch.from_file(path, shared=True, size=nbytes // 8, dtype=torch.float64).view(torch.complex128).view(shape)
        t.zero_()
        t._tilefft_path = path
        self.paths = getattr(self, "paths", []) + [path]
        return t

    def ipc_handle(self, t):
        return (t._tilefft_path, tuple(t.shape))

    def ipc_open(self, h):
        import torch
        path, shape = h
        nbytes = int(np.prod(shape)) * 16
        return torch.from_file(path, shared=True, size=nbytes // 8, dtype=torch.float64).view(torch.complex128)


def _p2p_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1707_07263_b200.distributed import DistributedFFT, column_slab
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle
    O = Oracle()
    ops = SharedMemOracleOps(n, world, rank)
    d = DistributedFFT(n, exchange="p2p", ops=ops)
    outs = []
    for seed in (11, 12, 13):  # three calls: both slabs of the double buffer, then the first again
        x = O.random_bench_signal(n, seed)
        outs.append(d.forward(torch.from_numpy(column_slab(x, world, rank))).numpy().copy())
    gathered = [None] * world
    dist.all_gather_object(gathered, outs)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    for path in ops.paths:
        os.unlink(path)
    dist.destroy_process_group()


def test_distributed_p2p_orchestration_gloo():
    """Peer-store exchange across 2 processes: every call matches the oracle,
    including back-to-back calls that alternate the two row slabs."""
    import multiprocessing as mp
    from paper_1707_07263_b200.distributed import assemble_output
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle, rel_l2
    n, world = 1 << 16, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = Oracle()
    for call, seed in enumerate((11, 12, 13)):
        got = assemble_output([gathered[r][call] for r in range(world)], n)
        assert rel_l2(got, O.fft_tiled(O.random_bench_signal(n, seed))) < 1e-12, call


def _worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1707_07263_b200.distributed import DistributedFFT, column_slab, shard_rows
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle
    O = Oracle()
    x = O.random_bench_signal(n, 11)
    d = DistributedFFT(n, exchange="nccl", ops=OracleOps(n, world, rank))
    out = d.forward(torch.from_numpy(column_slab(x, world, rank)))
    slabs = [None] * world
    dist.all_gather_object(slabs, out.numpy())
    # batch sharding covers every transform exactly once
    shares = [None] * world
    dist.all_gather_object(shares, shard_rows(10, world, rank))
    if rank == 0:
        q.put((slabs, shares))
    dist.destroy_process_group()


def test_distributed_four_step_orchestration_gloo():
    import multiprocessing as mp
    from paper_1707_07263_b200.distributed import assemble_output
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle, rel_l2
    n, world = 1 << 16, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    slabs, shares = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = assemble_output(slabs, n)
    O = Oracle()
    want = O.fft_tiled(O.random_bench_signal(n, 11))
    assert rel_l2(got, want) < 1e-12
    assert shares == [(0, 5), (5, 10)]


def _natural_worker(rank, world, port, n, exchange, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1707_07263_b200.distributed import DistributedFFT, natural_block
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle
    O = Oracle()
    ops = SharedMemOracleOps(n, world, rank) if exchange == "p2p" else OracleOps(n, world, rank)
    d = DistributedFFT(n, exchange=exchange, ops=ops)
    outs = []
    for seed in (21, 22):
        x = O.random_bench_signal(n, seed)
        outs.append(d.forward_natural(torch.from_numpy(natural_block(x, world, rank))).numpy().copy())
    gathered = [None] * world
    dist.all_gather_object(gathered, outs)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    for path in getattr(ops, "paths", []):
        os.unlink(path)
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_distributed_natural_order_io_gloo(exchange):
    """Natural-order block I/O (SURVEY §8e option): each rank passes its contiguous 1/G of x and gets its
    contiguous 1/G of X; the concatenation equals the oracle's transform."""
    import multiprocessing as mp
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle, rel_l2
    n, world = 1 << 16, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_natural_worker, args=(r, world, port, n, exchange, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = Oracle()
    for call, seed in enumerate((21, 22)):
        got = np.concatenate([gathered[r][call] for r in range(world)])
        assert rel_l2(got, O.fft_tiled(O.random_bench_signal(n, seed))) < 1e-12, call


def test_layout_helpers_roundtrip():
    from paper_1707_07263_b200.distributed import column_slab, four_step_layout, shard_rows
    n, world = 1 << 18, 4
    n1, n2, c, r = four_step_layout(n, world)
    assert n1 * n2 == n and c * world == n2 and r * world == n1
    x = np.arange(n)
    slabs = [column_slab(x, world, g) for g in range(world)]
    for g, s in enumerate(slabs):
        assert s.shape == (n1, c)
        assert s[3, 5] == g * c + 5 + n2 * 3
    spans = [shard_rows(65536, 3, g) for g in range(3)]
    assert spans[0][0] == 0 and spans[-1][1] == 65536
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.gpu
@pytest.mark.parametrize("n,world", [(1 << 20, 1), (1 << 20, 2), (1 << 22, 4), (1 << 22, 8)])
@pytest.mark.parametrize("exchange", ["p2p", "staging"])
def test_distributed_pass_kernels_virtual_ranks(oracle, n, world, exchange):
    """G virtual ranks on one B200: pass-1 scatters into G row slabs (the
    peer-store epilogue), then pass 2; bit-level layout + tolerance check."""
    import torch
    from paper_1707_07263_b200 import _capi
    from paper_1707_07263_b200.distributed import assemble_output, column_slab
    from oracle_lib import rel_l2
    x = oracle.random_bench_signal(n, 5).astype(np.complex64)
    plans = [_capi.DistPlan.create_dist(n, world, g, 8, 0) for g in range(world)]
    lay = plans[0].layout()
    n1, n2, c, r = lay["n1"], lay["n2"], lay["cols_per_rank"], lay["rows_per_rank"]
    rows = [torch.zeros((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)]
    stage = [torch.zeros((world, r, c), dtype=torch.complex64, device="cuda") for _ in range(world)]
    for g, p in enumerate(plans):
        if exchange == "p2p":
            p.set_peers([t.data_ptr() for t in rows], n2, g * c)
        else:
            p.set_peers([stage[g][d].data_ptr() for d in range(world)], c, 0)
    slabs = [torch.from_numpy(column_slab(x, world, g)).cuda() for g in range(world)]
    for g, p in enumerate(plans):
        p.pass1(slabs[g].data_ptr())
    torch.cuda.synchronize()
    if exchange == "staging":  # the all-to-all: block d of rank s -> rank d, columns s*C..
        for d in range(world):
            for s in range(world):
                rows[d][:, s * c:(s + 1) * c] = stage[s][d]
    outs = [torch.empty_like(rows[g]) for g in range(world)]
    for g, p in enumerate(plans):
        p.pass2(rows[g].data_ptr(), outs[g].data_ptr())
    torch.cuda.synchronize()
    got = assemble_output([o.cpu().numpy() for o in outs], n)
    want = oracle.fft_tiled(x)
    err = rel_l2(got, want)
    assert err <= 1e-5 * math.log2(n), err
    assert err < 5e-7


@pytest.mark.gpu
def test_distributed_inverse_roundtrip_virtual_ranks(oracle):
    import torch
    from paper_1707_07263_b200 import _capi
    from paper_1707_07263_b200.distributed import column_slab, assemble_output
    from oracle_lib import rel_l2
    n, world = 1 << 20, 2
    x = oracle.random_bench_signal(n, 6).astype(np.complex64)

    def run(sig, sign):
        plans = [_capi.DistPlan.create_dist(n, world, g, 8, 0) for g in range(world)]
        lay = plans[0].layout()
        n2, c, r = lay["n2"], lay["cols_per_rank"], lay["rows_per_rank"]
        rows = [torch.zeros((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)]
        for g, p in enumerate(plans):
            p.set_peers([t.data_ptr() for t in rows], n2, g * c)
        slabs = [torch.from_numpy(column_slab(sig, world, g)).cuda() for g in range(world)]
        for g, p in enumerate(plans):
            p.pass1(slabs[g].data_ptr(), sign)
        torch.cuda.synchronize()
        outs = [torch.empty_like(t) for t in rows]
        for g, p in enumerate(plans):
            p.pass2(rows[g].data_ptr(), outs[g].data_ptr(), sign)
        torch.cuda.synchronize()
        return assemble_output([o.cpu().numpy() for o in outs], n)

    X = run(x, _capi.FORWARD)
    want_inv = oracle.fft_tiled(X.astype(np.complex64), inverse=True)
    got_inv = run(X.astype(np.complex64), _capi.INVERSE)
    assert rel_l2(got_inv, want_inv) <= 1e-5 * 20
    assert rel_l2(got_inv, x) <= 1e-5 * 20


def _virtual_step_setup(n, world):
    """G virtual ranks on one B200 with two row slabs each and the device-barrier flags wired up."""
    import torch
    from paper_1707_07263_b200 import _capi
    plans = [_capi.DistPlan.create_dist(n, world, g, 8, 0) for g in range(world)]
    lay = plans[0].layout()
    n2, c, r = lay["n2"], lay["cols_per_rank"], lay["rows_per_rank"]
    slabs = [[torch.zeros((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)] for _ in range(2)]
    flags = [p.flag_buffer() for p in plans]
    for p in plans:
        p.set_flags(flags)
    streams = [torch.cuda.Stream() for _ in range(world)]
    return plans, slabs, streams, n2, c, r


@pytest.mark.gpu
@pytest.mark.parametrize("n,world", [(1 << 20, 2), (1 << 22, 4)])
def test_distributed_device_barrier_virtual_ranks(oracle, n, world):
    """tilefft_dist_exec (pass 1 -> peer-flag barrier kernel -> pass 2, no host sync) with every virtual rank on
    its own stream, three back-to-back calls alternating the two row slabs, each vs the oracle."""
    import torch
    from paper_1707_07263_b200.distributed import assemble_output, column_slab
    from oracle_lib import rel_l2
    plans, slabs, streams, n2, c, r = _virtual_step_setup(n, world)
    xs = [oracle.random_bench_signal(n, 20 + i).astype(np.complex64) for i in range(3)]
    ins = [[torch.from_numpy(column_slab(x, world, g)).cuda() for g in range(world)] for x in xs]
    outs = [[torch.empty((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)] for _ in xs]
    torch.cuda.synchronize()
    for i in range(3):
        b = i & 1
        for g, p in enumerate(plans):  # all calls queued without any host synchronisation
            p.set_peers([t.data_ptr() for t in slabs[b]], n2, g * c)
            p.exec_step(ins[i][g].data_ptr(), outs[i][g].data_ptr(), stream=streams[g].cuda_stream)
    torch.cuda.synchronize()
    for i, x in enumerate(xs):
        got = assemble_output([o.cpu().numpy() for o in outs[i]], n)
        err = rel_l2(got, oracle.fft_tiled(x))
        assert err < 5e-7, (i, err)


@pytest.mark.gpu
def test_distributed_step_graph_capture_virtual_ranks(oracle):
    """The distributed step is graph-capturable: each virtual rank's tilefft_dist_exec captured into a CUDA graph
    (one per slab parity) and replayed gives the directly executed result bit for bit."""
    import torch
    from paper_1707_07263_b200.distributed import assemble_output, column_slab
    from oracle_lib import rel_l2
    n, world = 1 << 20, 2
    plans, slabs, streams, n2, c, r = _virtual_step_setup(n, world)
    x = oracle.random_bench_signal(n, 31).astype(np.complex64)
    ins = [torch.from_numpy(column_slab(x, world, g)).cuda() for g in range(world)]
    direct = [torch.empty((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)]
    outs = [torch.empty((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)]
    for g, p in enumerate(plans):  # direct run (also creates the inner plans' graphs)
        p.set_peers([t.data_ptr() for t in slabs[0]], n2, g * c)
        p.exec_step(ins[g].data_ptr(), direct[g].data_ptr(), stream=streams[g].cuda_stream)
    for g, p in enumerate(plans):  # warm the (slab, out) pair the graphs will use
        p.set_peers([t.data_ptr() for t in slabs[1]], n2, g * c)
        p.exec_step(ins[g].data_ptr(), outs[g].data_ptr(), stream=streams[g].cuda_stream)
    torch.cuda.synchronize()
    graphs = []
    for g, p in enumerate(plans):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=streams[g]):
            p.set_peers([t.data_ptr() for t in slabs[1]], n2, g * c)
            p.exec_step(ins[g].data_ptr(), outs[g].data_ptr(), stream=streams[g].cuda_stream)
        graphs.append(gr)
    torch.cuda.synchronize()
    for rep in range(2):
        for g in range(world):
            with torch.cuda.stream(streams[g]):
                graphs[g].replay()
        torch.cuda.synchronize()
        for g in range(world):
            assert torch.equal(outs[g], direct[g]), (rep, g)
    got = assemble_output([o.cpu().numpy() for o in outs], n)
    assert rel_l2(got, oracle.fft_tiled(x)) < 5e-7


def _ipc_worker(rank, world, port, n, q, per_rank_gpu=False):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if per_rank_gpu else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1707_07263_b200.distributed import DistributedFFT, column_slab
    sys.path.insert(0, HERE)
    from oracle_lib import Oracle
    O = Oracle()
    d = DistributedFFT(n, exchange="p2p", device=dev)
    assert d.device_barrier
    outs = []
    for seed in (41, 42, 43):  # both slabs of the double buffer, then the first again
        x = O.random_bench_signal(n, seed).astype(np.complex64)
        y = d.forward(torch.from_numpy(column_slab(x, world, rank)).to(f"cuda:{dev}"))
        torch.cuda.synchronize()
        outs.append(y.cpu().numpy())
    gathered = [None] * world
    dist.all_gather_object(gathered, outs)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    d.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("per_rank_gpu", [False, True], ids=["same_gpu", "gpu_per_rank"])
def test_distributed_two_processes_cuda_ipc(oracle, per_rank_gpu):
    """Two real processes (gloo for the handle exchange, both on cuda:0): pass-1 stores land in the other process's
    row slab through CUDA IPC and the device flag barrier orders them — the cross-process path of the p2p exchange
    (on an 8-GPU box the same code maps peer GPUs' memory over NVLink)."""
    import multiprocessing as mp
    from paper_1707_07263_b200.distributed import assemble_output
    from oracle_lib import rel_l2
    import torch
    if per_rank_gpu and torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (peer memory over NVLink); the same-GPU case covers the protocol")
    n, world = 1 << 20, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, n, q, per_rank_gpu)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for call, seed in enumerate((41, 42, 43)):
        got = assemble_output([gathered[r][call] for r in range(world)], n)
        want = oracle.fft_tiled(oracle.random_bench_signal(n, seed).astype(np.complex64))
        assert rel_l2(got, want) < 5e-7, call


@pytest.mark.gpu
@pytest.mark.parametrize("n,world", [(1 << 24, 2), (1 << 24, 4), (1 << 26, 8)])
def test_distributed_pass2_reads_alltoall_blocks(oracle, n, world):
    """NCCL-exchange layout: pass 1 stages per-destination blocks, the all-to-all (simulated: rank d receives
    block d of every source) leaves [src][k1][c], and pass 2 reads that buffer through its 5-D tensor map
    (tilefft_dist_exec_pass2_blocks) -- no re-assembly copy; vs the oracle."""
    import torch
    from paper_1707_07263_b200 import _capi
    from paper_1707_07263_b200.distributed import assemble_output, column_slab
    from oracle_lib import rel_l2
    x = oracle.random_bench_signal(n, 7).astype(np.complex64)
    plans = [_capi.DistPlan.create_dist(n, world, g, 8, 0) for g in range(world)]
    lay = plans[0].layout()
    n2, c, r = lay["n2"], lay["cols_per_rank"], lay["rows_per_rank"]
    stage = [torch.zeros((world, r, c), dtype=torch.complex64, device="cuda") for _ in range(world)]
    for g, p in enumerate(plans):
        p.set_peers([stage[g][d].data_ptr() for d in range(world)], c, 0)
        p.pass1(torch.from_numpy(column_slab(x, world, g)).cuda().data_ptr())
    torch.cuda.synchronize()
    recv = [torch.stack([stage[s][d] for s in range(world)]).contiguous() for d in range(world)]
    outs = [torch.empty((r, n2), dtype=torch.complex64, device="cuda") for _ in range(world)]
    for d, p in enumerate(plans):
        p.pass2_blocks(recv[d].data_ptr(), outs[d].data_ptr())
    torch.cuda.synchronize()
    got = assemble_output([o.cpu().numpy() for o in outs], n)
    err = rel_l2(got, oracle.fft_tiled(x))
    assert err < 5e-7, err


@pytest.mark.gpu
def test_distributed_pass2_blocks_needs_multipass_rows(oracle):
    from paper_1707_07263_b200 import _capi
    p = _capi.DistPlan.create_dist(1 << 20, 2, 0, 8, 0)  # 1024-point rows: a single pass
    with pytest.raises(ValueError, match="single pass"):
        p.pass2_blocks(0x1000, 0x1000)
