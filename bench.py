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
}


# device pass factorisation each config's default plan executes (asserted by tests/test_gpu_bench_plans.py)
DEVICE_FACTORS = {
    "batched1024": [1024],
    "1d_2e20": [1024, 1024],
    "1d_2e26": [512, 512, 256],
    "2d_8192": [8192, 8192],
    "1d_2e30": [1024, 1024, 1024],
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
            "config": {"workload": desc, "n": n, "batch": batch, "kind": kind}}
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
        ctx = R.lib.ref_ctx_create(n, 1024) if R is not None else None
        run = (lambda: R.lib.ref_ctx_exec_batched(ctx, ctypes.c_void_p(x.ctypes.data),
                                                  ctypes.c_void_p(out.ctypes.data), rows, threads))
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
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="batched1024", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    from paper_1707_07263_b200 import _capi

    n, batch, kind, p_alg, desc = cfg
    total = n * n if kind == "2d" else n
    steps, warmup = args.steps, max(3, args.warmup)

    # ---- plan + resident input (synthetic, counter-based, per-rank seed)
    distributed = world > 1 and kind == "1d" and batch == 1
    if distributed:
        # one transform over all ranks: four-step, pass-1 store = the all-to-all
        from paper_1707_07263_b200.distributed import DistributedFFT
        dfft = DistributedFFT(total, exchange=args.exchange, device=dev)
        o = dfft.ops
        elems = o.n1 * o.c
        host_in = splitmix_signal(elems, seed=1 + rank)
        x = torch.from_numpy(host_in.view(np.float32)).to(f"cuda:{dev}").view(torch.complex64).view(o.n1, o.c)
        y = o.alloc((o.r, o.n2))
        info = {"passes": 1 + len(o.plan.info()["factors"]) - 1, "launches_per_exec": None,
                "factors": o.plan.info()["factors"]}
        stream = torch.cuda.current_stream()

        def step():
            dfft.forward(x, y)
    else:
        plan = make_device_plan(args.config, dev)
        info = plan.info()
        elems = total * batch
        host_in = splitmix_signal(elems, seed=1 + rank)
        x = torch.from_numpy(host_in.view(np.float32)).to(f"cuda:{dev}")
        y = torch.empty_like(x)
        stream = torch.cuda.current_stream()
        sptr = stream.cuda_stream

        def step():
            plan.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, sptr)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / steps
    flops_job = flops_per_transform(n, kind) * (1 if distributed else batch * world)
    value = flops_job / (ms_step * 1e-3) / 1e9

    # ---- dominant kernel: per-launch CUDA-event durations on the launching stream
    kernel_ms = []
    if info["passes"] == 1:
        kernel_ms = [ms_step]
    else:
        # time each pass separately by rebuilding a single-pass view is not exposed; use step time / passes
        kernel_ms = [ms_step]
    alg_bytes = p_alg * 2 * total * 8 * batch  # per launch == per step for single-pass plans
    if distributed:
        alg_bytes = p_alg * 2 * total * 8 // world  # this rank's share of the HBM traffic
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / (statistics.mean(kernel_ms) * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": profile_traffic(args.config),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_step": alg_bytes, "device_passes": info["passes"], "p_alg": p_alg}

    # ---- e2e through the C ABI host entry point, pinned host buffers
    e2e = None
    if args.e2e_steps > 0 and not distributed:
        hin = torch.from_numpy(host_in.view(np.float32)).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        if kind == "2d":
            hplan = plan
        else:
            hplan = _capi.DevicePlan.create(total, batch, None, 8, _capi.MODE_FAST, None, dev)
        hplan.exec_host(hin.data_ptr(), hout.data_ptr(), _capi.FORWARD)  # warm-up (allocs staging)
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            hplan.exec_host(hin.data_ptr(), hout.data_ptr(), _capi.FORWARD)
            ts.append(time.perf_counter() - t0)
        t_e2e = statistics.median(ts)
        if world > 1:
            t = torch.tensor([t_e2e], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        nbytes = elems * 8
        e2e = {"value": round(flops_job / t_e2e / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": round(t_e2e * 1e3, 3),
               "api": "tilefft_exec_c2c_host (pinned host buffers, 16 MiB chunks, H2D, kernel and D2H queues overlapped)"}

    # ---- CPU baseline: the reference itself on this host (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            r = cpu_reference_timing(n, batch, kind, threads, budget_s=args.ref_budget)
            cpu = {"value": round(r["value"], 3), "unit": "GFLOP/s", "cores": threads, "kind": r["kind"],
                   "sample": r["sample"]}
        except Exception as exc:  # report, never fail the GPU line
            cpu = {"value": None, "unit": "GFLOP/s", "cores": None, "kind": None, "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "C2C FFT GFLOP/s (5N*log2N/t)", "value": round(value, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "strong" if distributed else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (counter-based uniform(-1,1), per-rank seed)",
            "config": {"workload": desc, "n": n, "batch_per_gpu": batch, "kind": kind,
                       "parallelism": (f"four-step over {world} GPUs, {args.exchange} all-to-all fused into pass 1"
                                       if distributed else f"batch sharded over {world} GPU(s), no collective"),
                       "l2": "inputs larger than L2" if elems * 16 > 126 * 2 ** 20 else "L2-resident (no flush)",
                       "device_factors": info["factors"]},
            "hbm_gbs": round(achieved, 1),
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": steps * (info["launches_per_exec"] if info.get("launches_per_exec") else
                                     len(info["factors"])),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
