#!/usr/bin/env python
"""bench.py -- batched 1-D complex fp32 FFT on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (BASELINE.json configs[1]): N=4096, batch=65536 per GPU, split
re/im layout, forward.  A step is one execute of the whole batch.  Inputs
(2 GiB) and outputs (2 GiB) per GPU are far larger than the 126 MB L2, so no
flush is needed between steps.  Multi-GPU: the batch shards with no
communication (weak scaling, per-GPU batch fixed), timed per rank with CUDA
events and reduced with MAX.

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's
own CPU path (oracle/_ref: compile_pipeline + interpret, fp64) on the host's
cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched 1-D complex FFT GFLOP/s (5N log2N) and % of HBM roofline at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--layout", choices=["split", "interleaved"], default="split")
    ap.add_argument("--direction", choices=["forward", "inverse"], default="forward")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no JSON)")
    ap.add_argument("--workload", choices=["batched", "distributed"], default="batched",
                    help="distributed: one N-point transform over all ranks (config C5, e.g. --n 1073741824)")
    return ap.parse_args()


def gflop(n: int, batch: int) -> float:
    return 5.0 * n * math.log2(n) * batch / 1e9


def workload(a) -> dict:
    return {"workload": f"c2c fp32 FFT N={a.n} batch={a.batch}/GPU {a.layout} {a.direction}",
            "n": a.n, "batch_per_gpu": a.batch, "layout": a.layout, "direction": a.direction,
            "l2": "inputs+outputs (16N*batch = %.1f GiB/GPU) exceed the 126 MB L2; no flush"
                  % (16 * a.n * a.batch / 2 ** 30),
            "parallelism": f"batch-sharded x{a.gpus}, no collective"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region via NVML
    (B200_PROFILING.md clocks line); polls every 2 ms on a thread."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, dev: int):
        self.dev = dev
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._poll()  # one sample before the region starts
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # reported, not hidden
            self.nv = None
            self.err = str(e)
        return self

    def _poll(self):
        sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        reasons = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((sm, self.max_sm, reasons))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._poll()
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "t", None):
            self.t.join(timeout=1)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "error": getattr(self, "err", "no samples")}
        sms = [s[0] for s in self.samples]
        reasons = sorted({name for _, _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(sms)), "sm_max_mhz": float(self.samples[0][1]),
                "reasons": reasons, "samples": len(sms), "source": "nvml"}


# ------------------------------------------------------------ CPU legs
def cpu_reference_rate(a, budget_s: float, threads: int, with_aot: bool = True) -> dict:
    """The reference's own CPU path (compile_pipeline + interpret, fp64,
    oracle/_ref) batch-parallel over `threads` host cores on a bounded sample
    of the workload; GFLOP/s of 5N log2N."""
    import oracle
    if a.n > 65536:  # the interpreter needs ~46 s and 13 GB for one 2^24 transform
        return {"value": None, "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                "sample": f"skipped: N={a.n} > 2^16 is beyond a bounded CPU sample"}
    ref = oracle.Ref()
    alg, radix = "stockham", 4  # the reference's best interpreter config at N=4096
    lay = a.layout
    ref.compile(a.n, alg, radix, lay)
    chunk = max(threads * 4, 8)
    x = np.stack([ref.seeded_input(a.n, 1 + b) for b in range(chunk)])
    if lay == "split":
        x = oracle.relayout_to_split(x)
    x = x.astype(np.float32).astype(np.float64)
    done, t0 = 0, time.perf_counter()
    while True:
        ref.forward(x, alg, radix, lay, threads=threads)
        done += chunk
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    out = {"value": gflop(a.n, done) / el, "unit": "GFLOP/s", "cores": threads, "kind": "reference",
           "sample": f"{done} transforms of N={a.n} {lay} (fp32-rounded seeded_input), "
                     f"compile_pipeline(stockham, radix 4)+interpret fp64, {el:.1f} s wall, "
                     f"{threads} threads"}
    aot = cpu_aot_rate(a, x if lay == "split" else None, min(4.0, budget_s), threads) if with_aot else None
    if aot is not None:
        out["aot_emit_c"] = aot
    return out


def cpu_aot_rate(a, x_split, budget_s: float, threads: int):
    """The reference's ahead-of-time path (its emit_c output for this plan,
    compiled -O3, oracle/_ref/libref_aot.so) on the same sample: reported
    beside the interpreter, which is the reference's execute API."""
    import oracle
    if a.n != oracle.AotRef.N or a.layout != oracle.AotRef.LAYOUT or x_split is None:
        return None
    if not os.path.exists(oracle.AOT_SO):
        return {"value": None, "sample": "oracle/_ref/libref_aot.so not built"}
    aot = oracle.AotRef()
    xb = np.tile(x_split, (max(1, 4096 // x_split.shape[0]), 1))
    aot.forward(xb[:threads], threads)
    done, t0 = 0, time.perf_counter()
    while True:
        aot.forward(xb, threads)
        done += xb.shape[0]
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return {"value": gflop(a.n, done) / el, "unit": "GFLOP/s", "cores": threads, "kind": "reference",
            "sample": f"{done} transforms, the reference's emit_c output for (N={a.n}, stockham radix 4, "
                      f"split) compiled -O3 -march=x86-64-v3, _Thread_local scratch, {el:.1f} s wall, "
                      f"{threads} threads"}


def pcie_ceiling(h_src, h_dst, dev) -> float:
    """Concurrent pinned H2D + D2H copy bandwidth (GB/s, both directions
    summed): the ceiling of the e2e leg, which moves inputs in and results out."""
    import torch
    m = min(h_src.numel(), h_dst.numel(), (256 << 20) // h_src.element_size())
    src = h_src.reshape(-1)[:m]
    dst = h_dst.reshape(-1)[:m]
    d_a = torch.empty(m, dtype=h_src.dtype, device=dev)
    d_b = torch.empty(m, dtype=h_src.dtype, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(src, non_blocking=True)
        with torch.cuda.stream(s2):
            dst.copy_(d_b, non_blocking=True)

    both()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(4):
        both()
    torch.cuda.synchronize(dev)
    el = (time.perf_counter() - t0) / 4
    return round(2 * m * src.element_size() / el / 1e9, 1)


# ------------------------------------------------------------ our arm
def run_ours(a):
    import torch
    import torch.distributed as dist
    import paper_2308_00497_b200 as fg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)  # before NCCL init: each rank's communicator binds its own GPU
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, batch = a.n, a.batch
    direction = fg.FORWARD if a.direction == "forward" else fg.INVERSE
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=a.layout, batch=batch, device=local,
                                                 algorithm="stockham"))
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    if a.layout == "split":
        in0 = torch.rand(batch, n, device=dev, generator=g) * 2 - 1
        in1 = torch.rand(batch, n, device=dev, generator=g) * 2 - 1
        out0, out1 = torch.empty_like(in0), torch.empty_like(in1)
    else:
        in0 = torch.rand(batch, n, 2, device=dev, generator=g) * 2 - 1
        in1 = out1 = None
        out0 = torch.empty_like(in0)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.execute(in0, out0, in1, out1, direction=direction, stream=stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    if a.profile:
        return None

    # ---- timed region: K steps, one event pair per launch on the launching stream
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t_begin = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_begin.record(stream)
        for i in range(a.steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = t_begin.elapsed_time(t_end)
    kern_ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    t = torch.tensor([total_ms, kern_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_ms = float(t[0]), float(t[1])
    ms_per_step = total_ms / a.steps
    value = gflop(n, batch) * world / (ms_per_step / 1e3)

    # ---- e2e: public API with pinned HOST buffers (H2D + D2H inside every step)
    e2e = None
    if a.e2e_steps > 0:
        h_in0 = in0.cpu().pin_memory()
        h_out0 = torch.empty_like(h_in0).pin_memory()
        h_in1 = in1.cpu().pin_memory() if in1 is not None else None
        h_out1 = torch.empty_like(h_in1).pin_memory() if h_in1 is not None else None
        plan.execute_host(h_in0, h_out0, h_in1, h_out1, direction=direction)  # warm (staging alloc)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            plan.execute_host(h_in0, h_out0, h_in1, h_out1, direction=direction)
        el = torch.tensor([(time.perf_counter() - t0) / a.e2e_steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        nbytes = batch * n * 8
        pcie = pcie_ceiling(h_in0, h_out0, dev)
        moved = 2 * nbytes / float(el[0]) / 1e9
        e2e = {"value": gflop(n, batch) * world / float(el[0]), "unit": "GFLOP/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "ms_per_step": float(el[0]) * 1e3,
               "path": "fftgen_execute_host (C ABI), pinned host fp32, chunked H2D/kernel/D2H on 2 streams",
               "roofline": {"bound": "pcie", "achieved": round(moved, 1), "peak": pcie, "unit": "GB/s",
                            "frac": round(moved / pcie, 4) if pcie else None,
                            "peak_source": "measured in this run: concurrent pinned H2D + D2H copies (torch), "
                                           "256 MiB each way"}}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return None

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    alg_bytes = 16.0 * n * batch  # read + write fp32 complex once per transform
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            prof = json.load(f)
        traffic = prof.get(f"{a.layout}_{n}_{batch}", {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(a, a.cpu_seconds, os.cpu_count() or 1)
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "error": str(e)}

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: uniform [-1,1) re/im generated on device (torch.rand), resident in HBM",
        "config": workload(a),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": next((w for w in plan.describe().split() if "kernel<" in w), "?"),
                     "launches_per_step": plan.launches(), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "kernel_ms_avg": round(kern_ms, 4)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": a.steps * plan.launches(),
        "clocks": clk.summary(),
        "impl": "ours",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    import oracle
    if not os.path.exists(oracle.REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfftgen_ref.so not built"}))
        return None
    # each step = a bounded sample of the workload (the full 65536-transform
    # batch would take ~1 min per step on the interpreter)
    per_step = max(1.0, a.cpu_seconds / max(1, a.steps + a.warmup))
    for _ in range(a.warmup):
        cpu_reference_rate(a, per_step / 2, threads, with_aot=False)
    vals, samples = [], []
    for _ in range(a.steps):
        r = cpu_reference_rate(a, per_step, threads, with_aot=False)
        vals.append(r["value"])
        samples.append(r["sample"])
    v = float(np.mean(vals))
    # the reference's ahead-of-time C path on the same workload, reported beside it once
    aot = None
    if a.layout == "split":
        ref_x = None
        try:
            ref = oracle.Ref()
            ref_x = oracle.relayout_to_split(np.stack([ref.seeded_input(a.n, 1 + b) for b in range(64)]))
            ref_x = ref_x.astype(np.float32).astype(np.float64)
        except Exception:
            pass
        aot = cpu_aot_rate(a, ref_x, 4.0, threads)
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(gflop(a.n, a.batch) / v * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: fp32-rounded seeded_input (verify.cpp:69-78)", "config": workload(a),
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": samples[-1], "aot_emit_c": aot},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference = unmodified fftgen compile_pipeline+interpret (oracle/_ref), batch-parallel "
                "one transform per thread; ms_per_step extrapolated to the full batch",
    }
    print(json.dumps(line), flush=True)
    return line


def run_distributed(a):
    """Config C5: one N-point transform block-distributed over all ranks,
    three NCCL all-to-alls (paper_2308_00497_b200.distributed)."""
    import torch
    import torch.distributed as dist
    from paper_2308_00497_b200.distributed import DistributedFFT

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    dev = torch.device("cuda", local)
    n = a.n
    m = n // world
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    x = torch.complex(torch.rand(m, device=dev, generator=g) * 2 - 1, torch.rand(m, device=dev, generator=g) * 2 - 1)
    d = DistributedFFT(n, device=local)
    for _ in range(a.warmup):
        y = d.execute(x)
    torch.cuda.synchronize(dev)
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        s.record()
        for _ in range(a.steps):
            y = d.execute(x)
        e.record()
        torch.cuda.synchronize(dev)
    dist.barrier()
    t = torch.tensor([s.elapsed_time(e) / a.steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    del y
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(gflop(n, 1) / (ms / 1e3), 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: uniform [-1,1) re/im on device", "impl": "ours",
            "config": {"workload": f"single c2c fp32 FFT N={n} distributed over {world} GPU(s), "
                                   f"{d.n1}x{d.n2} four-step, 3 all-to-alls", "n": n, "n1": d.n1, "n2": d.n2},
            "clocks": clk.summary()}), flush=True)
    dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "distributed":
        run_distributed(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
