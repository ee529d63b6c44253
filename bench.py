#!/usr/bin/env python3
"""Benchmark of the B200 C2C FFT path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config NAME]

One JSON line on rank 0. A "step" is one pass of the hot path over one batch of
synthetic input: by default configs[1] of BASELINE.json, a batched 1D complex
fp32 FFT of N=1024 x 65536 transforms per GPU (weak scaling: every rank owns
its own batch; no collective on the data path).

* value      : GFLOP/s = 5 N log2 N x transforms / t, whole job, inputs already
               in HBM (CUDA events on the launching stream, max over ranks).
* e2e        : the same metric through the C ABI host entry point
               (tilefft_exec_c2c_host) from pinned host memory: H2D copy,
               passes and D2H copy of every transform inside the timed region.
* roofline   : dominant kernel, algorithmic bytes p_alg*2*N*8 per transform
               (memsim.hpp's 2*N*p law) / its average CUDA-event
               duration, against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline: the reference's own fft_tiled (oracle/_ref, compiled from the
               reference headers) on this host's cores, bounded sample.
* --impl reference: the reference's CPU path alone, on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, batch per GPU, kind, p_alg, description)
    "batched1024": (1024, 65536, "1d", 1,
                    "batched 1D complex fp32 forward FFT N=1024 x batch 65536 per GPU (BASELINE configs[1])"),
    "1d_2e20": (1 << 20, 1, "1d", 2, "single 1D complex fp32 forward FFT N=2^20 (BASELINE configs[0])"),
    "1d_2e26": (1 << 26, 1, "1d", 2, "single 1D complex fp32 forward FFT N=2^26 (BASELINE configs[2])"),
    "2d_8192": (8192, 1, "2d", 2, "2D complex fp32 forward FFT 8192x8192, one image per GPU (BASELINE configs[3])"),
    "1d_2e30": (1 << 30, 1, "1d", 3, "single 1D complex fp32 forward FFT N=2^30 on one GPU (BASELINE configs[4])"),
    "1d_2e30_natural": (1 << 30, 1, "1d", 3, "distributed 1D complex fp32 forward FFT N=2^30 with natural-order "
                        "block I/O (SURVEY 8e option: one all-to-all before and one after the four-step exchange)"),
}


# device pass factorisation each config's default plan executes (asserted by tests/test_gpu_bench_plans.py)
DEVICE_FACTORS = {
    "batched1024": [1024],
    "1d_2e20": [1024, 1024],
    "1d_2e26": [512, 512, 256],
    "2d_8192": [8192, 8192],
    "1d_2e30": [1024, 1024, 1024],
    "1d_2e30_natural": [1024, 1024, 1024],
}


def splitmix_signal(count: int, seed: int = 1) -> np.ndarray:
    """Counter-based uniform(-1,1) complex64 input; identical to
    the oracle's orc_splitmix_signal_f32, vectorised."""
    with np.errstate(over="ignore"):
        key = np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
        out = np.empty(2 * count, dtype=np.float32)
        chunk = 1 << 24
        for s in range(0, 2 * count, chunk):
            i = np.arange(s, min(2 * count, s + chunk), dtype=np.uint64)
            z = key + i + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            out[s:s + len(i)] = (u * 2.0 - 1.0).astype(np.float32)
    return out.view(np.complex64)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profile_traffic(config: str):
    """DRAM bytes (ncu dram__bytes_read + dram__bytes_write) per step from the committed launch lists
    (profiles/r01_launches_*_s3.csv): the one launch for single-pass plans, the sum over one step's
    passes for multi-pass plans (matching `achieved`, which is per step)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period_s: float = 0.002):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self._ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def flops_per_transform(n: int, kind: str) -> float:
    total = n * n if kind == "2d" else n
    return 5.0 * total * math.log2(total)


def make_device_plan(config: str, device: int = 0, batch=None):
    """The plan bench.py times for `config` (tests/test_gpu_bench_plans.py pins its parity)."""
    from paper_1707_07263_b200 import _capi
    n, b, kind, _, _ = CONFIGS[config]
    b = b if batch is None else batch
    if kind == "2d":
        return _capi.DevicePlan.create_2d(n, n, b, 8, device)
    return _capi.DevicePlan.create(n, b, None, 8, _capi.MODE_FAST, None, device)


# ---------------------------------------------------------------------------------------------------
def run_reference(args, cfg):
    """`--impl reference`: the reference's own CPU fft_tiled (oracle/_ref) on all host threads."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    n, batch, kind, p_alg, desc = cfg
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Reference, available_reference, Oracle  # CPU baseline leg only
    threads = os.cpu_count() or 1
    line = {"impl": "reference", "metric": "C2C FFT GFLOP/s (5N*log2N/t)", "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_key(args.config)}
    res = cpu_reference_timing(n, batch, kind, threads, budget_s=args.ref_budget, steps=args.steps,
                               warmup=args.warmup)
    line.update({"value": res["value"], "ms_per_step": res["ms_per_step"],
                 "cpu_baseline": {"value": res["value"], "unit": "GFLOP/s", "cores": threads,
                                  "kind": res["kind"], "sample": res["sample"]},
                 "e2e": {"value": res["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def cpu_reference_timing(n, batch, kind, threads, budget_s=12.0, steps=None, warmup=1):
    """Time the reference's fft_tiled on host cores. Each step is a bounded
    sample of the workload (a subset of the transforms, or the whole transform
    for single-transform configs); reports GFLOP/s on what was run."""
    import ctypes
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Reference, available_reference, Oracle
    if available_reference():
        R = Reference()
        kind_s = "reference"
    else:
        R = None
        kind_s = "port"
    fl = flops_per_transform(n, kind)
    if kind == "1d" and batch > 1:
        # batched: threads x fft_tiled(threads=1) over a strided subset of rows;
        # a step is the whole batch (capped at 65536 transforms)
        sample = min(batch, 65536)
        x = splitmix_signal(n * sample).reshape(sample, n)
        out = np.zeros_like(x)  # touched: no first-touch page faults inside the timed steps
        if R is not None:
            ctx = R.lib.ref_ctx_create(n, 1024)
            run = lambda: R.lib.ref_ctx_exec_batched(ctx, ctypes.c_void_p(x.ctypes.data),
                                                     ctypes.c_void_p(out.ctypes.data), sample, threads)
        else:
            O = Oracle()
            run = lambda: O.fft_tiled(x)
        units, what = sample, f"{sample} of {batch} transforms per step, {threads} std::threads x fft_tiled(threads=1)"
    elif kind == "1d":
        x = splitmix_signal(n)
        out = np.zeros_like(x)
        if R is not None:
            ctx = R.lib.ref_ctx_create(n, 1024)
            run = lambda: R.lib.ref_ctx_exec_single(ctx, ctypes.c_void_p(x.ctypes.data),
                                                    ctypes.c_void_p(out.ctypes.data), threads)
        else:
            O = Oracle()
            run = lambda: O.fft_tiled(x)
        units, what = 1, f"whole transform, fft_tiled(threads={threads}), make_plan(N, 1024)"
    else:  # 2d: rows then columns, bounded to a band of rows + matching columns work
        rows = min(n, max(threads * 16, 512))
        x = splitmix_signal(n * rows).reshape(rows, n)
        out = np.zeros_like(x)
        if R is not None:
            ctx = R.lib.ref_ctx_create(n, 1024)
            run = lambda: R.lib.ref_ctx_exec_batched(ctx, ctypes.c_void_p(x.ctypes.data),
                                                     ctypes.c_void_p(out.ctypes.data), rows, threads)
        else:
            O = Oracle()
            run = lambda: O.fft_tiled(x)
        fl = 5.0 * n * math.log2(n)  # per row transform
        units = rows
        what = (f"{rows} length-{n} row transforms per step ({threads} threads); 2D = 2*{n} such transforms "
                f"per image")
    t_w = time.perf_counter()
    k_w = 0
    while k_w < max(1, warmup) or time.perf_counter() - t_w < 1.0:  # >= 1 s of warm-up (threads, caches, pages)
        run()
        k_w += 1
    times = []
    t_start = time.perf_counter()
    k = 0
    while True:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
        k += 1
        if steps is not None and k >= steps:
            break
        if time.perf_counter() - t_start > budget_s and k >= 3:
            break
    t = statistics.median(times)
    return {"value": fl * units / t / 1e9, "ms_per_step": t * 1e3, "kind": kind_s,
            "sample": what + f"; median of {len(times)} steps"}


# ---------------------------------------------------------------------------------------------------
def device_input(torch, elems: int, seed: int, dev: int):
    """Synthetic input resident in HBM (interleaved fp32 pairs): the counter-based splitmix64 signal
    (identical to the oracle's orc_splitmix_signal_f32) up to 2^27 complex elements; above that a seeded
    torch Philox uniform(-1,1) drawn on the device (generating 2^30 points in numpy would take ~1 min)."""
    if elems <= (1 << 27):
        return torch.from_numpy(splitmix_signal(elems, seed=seed).view(np.float32)).to(f"cuda:{dev}")
    g = torch.Generator(device=f"cuda:{dev}")
    g.manual_seed(seed)
    x = torch.empty(2 * elems, dtype=torch.float32, device=f"cuda:{dev}")
    x.uniform_(-1.0, 1.0, generator=g)
    return x


def config_key(name: str) -> dict:
    """The workload description both arms (b200 and --impl reference) print identically."""
    n, batch, kind, _, desc = CONFIGS[name]
    elems = (n * n if kind == "2d" else n) * batch
    return {"workload": desc, "name": name, "n": n, "batch_per_gpu": batch, "kind": kind,
            "l2": ("inputs larger than L2 (no flush needed)" if elems * 8 > 126 * 2 ** 20
                   else "L2-resident input: L2 flushed (256 MiB memset) before every timed step")}


class L2Flush:
    """Write a buffer larger than the 126 MB L2 between timed steps (L2-resident configs only)."""

    def __init__(self, torch, dev):
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    def __call__(self):
        self.buf.zero_()


def max_over_ranks(torch, dist, v: float, dev: int) -> float:
    """MAX of a per-rank scalar over the job (a CUDA tensor for NCCL, a host tensor for gloo)."""
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{dev}" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_steps(torch, step, stream, steps, flush=None):
    """Device time per step (ms): CUDA events on the launching stream around the K steps; with an L2 flush,
    events bracket each step so the flush itself is not counted."""
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush()
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / steps


def cufft_timing(torch, name, x, steps, warmup, flush):
    """torch.fft (cuFFT) on the same resident input, same event method: a comparison column, off the product path."""
    n, batch, kind, _, _ = CONFIGS[name]
    xc = x.view(torch.complex64)
    if kind == "2d":
        xc = xc.view(batch, n, n)
        f = lambda: torch.fft.fft2(xc)
    else:
        xc = xc.view(batch, n)
        f = lambda: torch.fft.fft(xc, dim=-1)
    try:
        for _ in range(max(3, warmup)):
            f()
        torch.cuda.synchronize()
        ms = time_steps(torch, f, torch.cuda.current_stream(), steps, flush)
        return {"ms_per_step": round(ms, 5), "value": round(flops_per_transform(n, kind) * batch / (ms * 1e-3) / 1e9, 2),
                "unit": "GFLOP/s", "api": "torch.fft (cuFFT), comparison only, same CUDA-event method"}
    except Exception as exc:  # comparison only: never fail the line
        return {"ms_per_step": None, "value": None, "unit": "GFLOP/s", "api": f"torch.fft failed: {exc}"}
    finally:
        torch.cuda.empty_cache()


def bench_config(name, args, torch, dev, world, rank, steps, warmup, with_cpu, with_cufft):
    """One config on this rank: device-resident step time, per-pass kernel times, roofline, e2e, cpu_baseline."""
    import torch.distributed as dist
    from paper_1707_07263_b200 import _capi
    n, batch, kind, p_alg, desc = CONFIGS[name]
    total = n * n if kind == "2d" else n
    distributed = world > 1 and kind == "1d" and batch == 1
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    plan = None
    if distributed:
        # one transform over all ranks: four-step, pass-1 store = the all-to-all
        from paper_1707_07263_b200.distributed import DistributedFFT
        dfft = DistributedFFT(total, exchange=args.exchange, device=dev)
        o = dfft.ops
        elems = o.n1 * o.c
        natural = name.endswith("_natural")
        x = device_input(torch, elems, 1 + rank, dev).view(torch.complex64).view(o.n1, o.c)
        y = o.alloc((o.r, o.n2))
        if natural:  # this rank's contiguous 1/G of the signal in, its contiguous 1/G of the spectrum out
            x = x.reshape(-1)
        fac = o.plan.info()["factors"]  # [N1] + the local row plan's passes
        info = {"passes": len(fac), "factors": fac,
                "launches_per_exec": len(fac) + (1 if getattr(dfft, "device_barrier", False) else 0)}

        def step():
            if natural:
                dfft.forward_natural(x)
            else:
                dfft.forward(x, y)
    else:
        plan = make_device_plan(name, dev)
        info = plan.info()
        elems = total * batch
        x = device_input(torch, elems, 1 + rank, dev)
        y = torch.empty_like(x)

        def step():
            plan.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, sptr)

    flush = L2Flush(torch, dev) if elems * 8 <= 126 * 2 ** 20 else None
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ms_step = time_steps(torch, step, stream, steps, flush)
    if world > 1:
        ms_step = max_over_ranks(torch, dist, ms_step, dev)
        dist.barrier()
    flops_job = flops_per_transform(n, kind) * (1 if distributed else batch * world)
    value = flops_job / (ms_step * 1e-3) / 1e9

    # ---- per-kernel durations: CUDA events between the plan's passes on the launching stream
    peak, peak_kind = measured_peaks()
    step_bytes = p_alg * 2 * total * 8 * batch  # algorithmic bytes of one step, this rank
    if distributed:
        step_bytes //= world
    pass_ms = None
    if plan is not None:
        if flush is None:
            pass_ms = plan.exec_timed(x.data_ptr(), y.data_ptr(), _capi.FORWARD, sptr, reps=max(3, min(steps, 20)))
        else:  # L2-resident: one flushed execution per sample
            acc = None
            reps = max(3, min(steps, 20))
            for _ in range(reps):
                flush()
                t = plan.exec_timed(x.data_ptr(), y.data_ptr(), _capi.FORWARD, sptr, reps=1)
                acc = t if acc is None else [a + b for a, b in zip(acc, t)]
            pass_ms = [a / reps for a in acc]
    if pass_ms:
        dom = max(range(len(pass_ms)), key=lambda i: pass_ms[i])
        kernel_bytes = 2 * total * 8 * batch  # every pass reads and writes each element once
        achieved = kernel_bytes / (pass_ms[dom] * 1e-3) / 1e9
        dominant = {"pass": dom, "length": info["factors"][dom] if dom < len(info["factors"]) else None,
                    "ms": round(pass_ms[dom], 5), "algorithmic_bytes": kernel_bytes}
    else:  # distributed: the whole step on this rank
        achieved = step_bytes / (ms_step * 1e-3) / 1e9
        dominant = {"pass": None, "ms": round(ms_step, 5), "algorithmic_bytes": step_bytes}
    nvlink = None
    if distributed:
        # pass 1 alone (its epilogue IS the all-to-all): remote bytes / pass-1 time, max over ranks
        reps = max(3, min(steps, 20))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            o.pass1(x.view(o.n1, o.c), _capi.FORWARD)
        b.record(stream)
        torch.cuda.synchronize()
        p1_ms = max_over_ranks(torch, dist, a.elapsed_time(b) / reps, dev)
        dist.barrier()
        remote = (world - 1) * (o.n1 // world) * o.c * 8  # rows of this rank's pass-1 output owned by peers
        nvlink = {"bytes_out_per_rank": remote, "pass1_ms": round(p1_ms, 5),
                  "nvlink_gbs": round(remote / (p1_ms * 1e-3) / 1e9, 1),
                  "peak_per_direction_gbs": 900.0, "exchange": args.exchange,
                  "note": "pass-1 kernel time with the all-to-all fused into its stores (p2p), max over ranks"
                          if args.exchange == "p2p" else "pass 1 + staging only; the NCCL all_to_all is separate"}
    traffic = profile_traffic(name)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": (None if distributed else traffic.get("dominant") if isinstance(traffic, dict)
                            else traffic if info["passes"] == 1 else None),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "dominant_kernel": dominant,
                "pass_ms": [round(v, 5) for v in pass_ms] if pass_ms else None,
                "step": {"algorithmic_bytes": step_bytes, "p_alg": p_alg, "device_passes": info["passes"],
                         "achieved": round(step_bytes / (ms_step * 1e-3) / 1e9, 1),
                         "frac": round(step_bytes / (ms_step * 1e-3) / 1e9 / peak, 4),
                         "traffic": (None if distributed else traffic.get("step") if isinstance(traffic, dict)
                                     else traffic)}}

    # ---- e2e through the C ABI host entry point, pinned host buffers
    e2e = None
    if args.e2e_steps > 0 and not distributed:
        hin = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        hin.copy_(x)
        hout = torch.empty_like(hin, pin_memory=True)
        plan.exec_host(hin.data_ptr(), hout.data_ptr(), _capi.FORWARD)  # warm-up (allocates staging)
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(args.e2e_steps if total * batch <= (1 << 27) else 2):
            t0 = time.perf_counter()
            plan.exec_host(hin.data_ptr(), hout.data_ptr(), _capi.FORWARD)
            ts.append(time.perf_counter() - t0)
        t_e2e = statistics.median(ts)
        if world > 1:
            t_e2e = max_over_ranks(torch, dist, t_e2e, dev)
        nbytes = elems * 8
        chunked = batch > 1 and info["passes"] == 1 and kind == "1d"
        e2e = {"value": round(flops_job / t_e2e / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": round(t_e2e * 1e3, 3),
               "api": ("tilefft_exec_c2c_host (pinned host buffers, 32 MiB chunks, H2D, kernel and D2H queues "
                       "overlapped)" if chunked else
                       "tilefft_exec_c2c_host (pinned host buffers; whole-transform H2D, passes, D2H)")}
        del hin, hout

    cufft = cufft_timing(torch, name, x, min(steps, 50), warmup, flush) if with_cufft and not distributed else None

    # ---- CPU baseline: the reference itself on this host (rank 0, N=1 only)
    cpu = None
    if with_cpu and rank == 0 and world == 1:
        if name == "1d_2e30" and not args.cpu_2e30:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": None, "kind": None,
                   "sample": "skipped by default (one reference fft_tiled of 2^30 takes ~1 min of host time and "
                             "16 GB of host memory); bench.py --cpu-2e30 runs it"}
        else:
            try:
                threads = os.cpu_count() or 1
                r = cpu_reference_timing(n, batch, kind, threads, budget_s=args.ref_budget)
                cpu = {"value": round(r["value"], 3), "unit": "GFLOP/s", "cores": threads, "kind": r["kind"],
                       "sample": r["sample"]}
            except Exception as exc:  # report, never fail the GPU line
                cpu = {"value": None, "unit": "GFLOP/s", "cores": None, "kind": None, "sample": f"failed: {exc}"}

    rec = {"value": round(value, 2), "unit": "GFLOP/s", "ms_per_step": round(ms_step, 5), "steps": steps,
           "warmup": warmup, "scaling": "strong" if distributed else "weak", "config": config_key(name),
           "parallelism": (f"four-step over {world} GPUs, {args.exchange} all-to-all fused into pass 1"
                           + (", natural-order block I/O (+2 NCCL all-to-alls)" if name.endswith("_natural") else "")
                           if distributed else f"batch sharded over {world} GPU(s), no collective"),
           "device_factors": info["factors"], "hbm_gbs": round(step_bytes / (ms_step * 1e-3) / 1e9, 1),
           "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "cufft": cufft, "nvlink": nvlink,
           "gpu_launches": steps * (info["launches_per_exec"] if info.get("launches_per_exec") else
                                    len(info["factors"])),
           "clocks": clk.summary()}
    del x, y
    if plan is not None:
        plan.close()
    if distributed:
        dfft.close()
    torch.cuda.empty_cache()
    return rec


SUB_STEPS = {"1d_2e20": 200, "1d_2e26": 100, "2d_8192": 100, "1d_2e30": 20}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="batched1024", choices=sorted(CONFIGS))
    ap.add_argument("--configs", default=None,
                    help="comma list of extra configs timed in the same process as sub-records "
                         "(default with --config batched1024: every other BASELINE config at N=1, 2d_8192 at N>1; "
                         "'none' to skip)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cufft", action="store_true")
    ap.add_argument("--cpu-2e30", action="store_true", help="also time the reference CPU fft_tiled at 2^30")
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="distributed single-transform configs at N>1: fused peer-store or NCCL all-to-all")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world > 1:
        # TILEFFT_BENCH_BACKEND=gloo + TILEFFT_BENCH_DEVICE=0: functional check of the N>1 path with every
        # rank on one GPU (NCCL refuses duplicate GPUs); timing such a run means nothing
        dev_idx = int(os.environ.get("TILEFFT_BENCH_DEVICE", local))
        torch.cuda.set_device(dev_idx)
        backend = os.environ.get("TILEFFT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    steps, warmup = args.steps, max(3, args.warmup)

    if args.configs is None:
        subs = ([c for c in ("1d_2e20", "1d_2e26", "2d_8192", "1d_2e30") if c != args.config]
                if args.config == "batched1024" and world == 1 else
                (["2d_8192", "1d_2e30", "1d_2e30_natural"] if args.config == "batched1024" else []))
    else:
        subs = [] if args.configs == "none" else [c for c in args.configs.split(",") if c and c != args.config]
    with_cpu = not args.no_cpu_baseline
    head = bench_config(args.config, args, torch, dev, world, rank, steps, warmup, with_cpu, not args.no_cufft)
    sub_recs = {}
    for c in subs:
        try:
            sub_recs[c] = bench_config(c, args, torch, dev, world, rank, min(steps, SUB_STEPS.get(c, steps)),
                                       warmup, with_cpu, not args.no_cufft)
        except Exception as exc:  # a sub-record never takes the headline down
            sub_recs[c] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {"metric": "C2C FFT GFLOP/s (5N*log2N/t)", "value": head["value"], "unit": "GFLOP/s",
                "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": head["ms_per_step"],
                "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None, "dtype": "f32",
                "data": ("synthetic uniform(-1,1), per-rank seed: counter-based splitmix64 up to 2^27 points, "
                         "device Philox above")}
        for k in ("config", "parallelism", "device_factors", "hbm_gbs", "roofline", "e2e", "cpu_baseline", "cufft",
                  "nvlink", "gpu_launches", "clocks"):
            line[k] = head[k]
        if sub_recs:
            line["configs"] = sub_recs
            line["gpu_launches"] = head["gpu_launches"] + sum(r.get("gpu_launches", 0) for r in sub_recs.values())
            line["gpu_launches_note"] = "headline + every sub-record's timed steps"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
