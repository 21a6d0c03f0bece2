#!/usr/bin/env python
"""bench.py -- batched 1-D complex fp32 FFT on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

`--gpus N` without a torchrun environment re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU); under
torchrun WORLD_SIZE must equal N.

Workload (BASELINE.json configs[1]): N=4096, batch=65536 per GPU, split
re/im layout, forward, on the reference's own inputs (seeded_input,
verify.cpp:55-78, transform b of rank r seeded 1 + r*batch + b) generated on
the device.  A step is one execute of the whole batch.  Inputs
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
    ap.add_argument("--order", choices=["natural", "cyclic"], default="natural",
                    help="distributed: output order (cyclic = X[rank + P j], two exchanges instead of three)")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="distributed: NCCL all-to-alls, or the exchanges fused into the kernels over symmetric memory")
    ap.add_argument("--launch-selftest", action="store_true",
                    help="CPU check of the rank launcher: gloo ranks all-reduce MAX of their rank")
    return ap.parse_args()


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_if_needed(a) -> bool:
    """`--gpus N` outside torchrun: re-exec this command as N torchrun ranks
    (the driver's own launch line).  Returns True when this process only
    launched the ranks."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != a.gpus:
            sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={env_world}")
        return False
    if a.gpus <= 1:
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)
    return True


def launch_selftest(a):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank), 1.0])
    if world > 1:
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
    if rank == 0:
        print(json.dumps({"selftest": "launch", "n_gpus": world, "max_rank": int(t[0]), "ranks": int(t[1]),
                          "gpus_flag": a.gpus}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def gflop(n: int, batch: int) -> float:
    return 5.0 * n * math.log2(n) * batch / 1e9


def workload(a, world: int = 1) -> dict:
    return {"workload": f"c2c fp32 FFT N={a.n} batch={a.batch}/GPU {a.layout} {a.direction}",
            "n": a.n, "batch_per_gpu": a.batch, "global_batch": a.batch * world, "layout": a.layout,
            "direction": a.direction,
            "l2": "inputs+outputs (16N*batch = %.1f GiB/GPU) exceed the 126 MB L2; no flush"
                  % (16 * a.n * a.batch / 2 ** 30),
            "parallelism": f"batch-sharded over {world} rank(s), no collective"}


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
    # the reference's inputs (seeded_input, verify.cpp:55-78), generated on the device
    seed0 = 1 + rank * batch
    if a.layout == "split":
        in0, in1 = fg.seeded_input(n, batch, "split", seed0=seed0, device=local)
        out0, out1 = torch.empty_like(in0), torch.empty_like(in1)
    else:
        in0 = fg.seeded_input(n, batch, "interleaved", seed0=seed0, device=local)
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

    if e2e and cpu and cpu.get("value"):
        # the end-to-end speed-up against both of the reference's CPU paths on
        # this host: its execute API (interpret, the reference arm) and its
        # ahead-of-time emitted C for the same plan (the faster, honest one)
        aot = (cpu.get("aot_emit_c") or {}).get("value")
        e2e["vs_cpu"] = {"reference_interpret": round(e2e["value"] / cpu["value"], 1),
                         "reference_emit_c": round(e2e["value"] / aot, 2) if aot else None}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: the reference's seeded_input (verify.cpp:55-78, splitmix64 uniform [-1,1) re/im), "
                "transform b of rank r seeded 1 + r*batch + b, generated on the device "
                "(fftgen_seeded_input), resident in HBM",
        "config": workload(a, world),
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
    """The reference arm: the unmodified reference (oracle/_ref, compiled from
    /root/reference's own sources) through its execute API
    (compile_pipeline + interpret, fp64), batch-parallel on all host cores.
    Each step is a MEASURED pass over a fixed sample of the workload's
    transforms (sample_transforms, sized from a calibration pass so a step
    takes ~2 s and the whole --steps/--warmup run a few minutes)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    import oracle
    if not os.path.exists(oracle.REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfftgen_ref.so not built"}))
        return None
    if a.n > 65536:
        print(json.dumps({"impl": "reference", "unavailable": f"N={a.n}: the reference interpreter needs ~46 s "
                                                              "and 13 GB per 2^24 transform (SURVEY 6)"}))
        return None
    ref = oracle.Ref()
    alg, radix, lay = "stockham", 4, a.layout  # the reference's best interpreter config at N=4096
    ref.compile(a.n, alg, radix, lay)
    chunk = max(threads * 4, 8)
    x = np.stack([ref.seeded_input(a.n, 1 + b) for b in range(chunk)])
    if lay == "split":
        x = oracle.relayout_to_split(x)
    x = x.astype(np.float32).astype(np.float64)
    # calibration: transforms per step for ~step_s seconds
    step_s = max(0.5, min(2.5, 120.0 / max(1, a.steps + a.warmup)))
    t0 = time.perf_counter()
    ref.forward(x, alg, radix, lay, threads=threads)
    rate = chunk / (time.perf_counter() - t0)
    calls = max(1, int(round(rate * step_s / chunk)))
    sample = calls * chunk

    def step():
        for _ in range(calls):
            ref.forward(x, alg, radix, lay, threads=threads)

    for _ in range(a.warmup):
        step()
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = float(np.mean(times)) * 1e3
    v = gflop(a.n, sample) / (ms / 1e3)
    # the reference's ahead-of-time C path on the same workload, reported beside it once
    aot = None
    if lay == "split":
        aot = cpu_aot_rate(a, x, 4.0, threads)
    cfg = workload(a, 1)
    cfg["sample_transforms"] = sample
    cfg["parallelism"] = f"host CPU, {threads} threads, one transform per thread"
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s", "n_gpus": 0, "launched_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: fp32-rounded seeded_input (verify.cpp:55-78)", "config": cfg,
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} transforms of N={a.n} {lay} per step (seeds 1..{chunk}, repeated), "
                                   f"compile_pipeline(stockham, radix 4)+interpret fp64, measured per step",
                         "aot_emit_c": aot},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference = unmodified fftgen compile_pipeline+interpret (oracle/_ref) on the host cores, "
                "batch-parallel one transform per thread; each step is a measured pass over "
                "config.sample_transforms transforms of the workload (n_gpus 0: no GPU on this path)",
    }
    print(json.dumps(line), flush=True)
    return line


def a2a_probe(m: int, dev, world: int, reps: int = 10) -> dict:
    """all_to_all_single (NCCL grouped send/recv) of an m-element complex64
    block per rank: the exchange roofline of the distributed four-step."""
    import torch
    import torch.distributed as dist
    send = torch.empty(m, dtype=torch.complex64, device=dev).uniform_()
    recv = torch.empty_like(send)

    def xchg():
        if world == 1:
            recv.copy_(send)
        else:
            dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send))

    for _ in range(3):
        xchg()
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        xchg()
    e.record()
    torch.cuda.synchronize(dev)
    t = torch.tensor([s.elapsed_time(e) / reps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    wire = 8 * m * (world - 1) / world if world > 1 else 16 * m  # bytes leaving each GPU / HBM bytes of the copy
    return {"ms": ms, "gbs": wire / (ms / 1e3) / 1e9,
            "what": ("all_to_all_single over NCCL, bytes sent per GPU / time" if world > 1
                     else "world 1: the exchange is a device copy (HBM read + write bytes / time)")}


def run_distributed(a):
    """Config C5: one N-point transform block-distributed over all ranks:
    exchange -> butterfly -> exchange -> local -> exchange -> unpack
    (paper_2308_00497_b200.distributed.DistributedFFT)."""
    import torch
    import torch.distributed as dist
    import paper_2308_00497_b200 as fg
    from paper_2308_00497_b200.distributed import DistributedFFT

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    n = a.n
    m = n // world
    # rank r's block of the reference input x = seeded_input(n, 1), generated on the device
    x = torch.view_as_complex(fg.seeded_input(n, 1, "interleaved", seed0=1, device=local)[0][rank * m:(rank + 1) * m])
    x = x.contiguous()
    d = DistributedFFT(n, device=local, transport=a.transport, output_order=a.order)
    cyclic = a.order == "cyclic" and world > 1
    if a.transport == "p2p":
        d.input_block().copy_(x)
        x = d.input_block()  # zero-copy input: the symmetric block itself
    out = torch.empty_like(x)
    direction = fg.FORWARD if a.direction == "forward" else fg.INVERSE
    for _ in range(a.warmup):
        d.execute(x, direction, out=out)
    torch.cuda.synchronize(dev)
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        s.record()
        for _ in range(a.steps):
            d.execute(x, direction, out=out)
        e.record()
        torch.cuda.synchronize(dev)
    dist.barrier()
    t = torch.tensor([s.elapsed_time(e) / a.steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    # per-stage device times of one execute (events between the stages)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    if a.transport == "p2p":
        names = ["barrier1", "butterfly+exchanges1,2", "barrier2", "local", "barrier3", "unpack+exchange3"]
        xb, rb, zb = d._blocks[0], d._blocks[1], d._blocks[2]
        ev[0].record()
        d._barrier(); ev[1].record()
        d.stages.butterfly_peers(d._peer["x"], d._peer["recv"], direction); ev[2].record()
        d._barrier(); ev[3].record()
        d.stages.local(rb, out if cyclic else zb, direction); ev[4].record()
        if cyclic:
            ev[5].record(); ev[6].record()
        else:
            d._barrier(); ev[5].record()
            d.stages.unpack_peers(d._peer["z"], out); ev[6].record()
            d._barrier()
    else:
        names = ["exchange1", "butterfly", "exchange2", "local", "exchange3", "unpack"]
        if world == 1:
            w0, w1 = torch.empty_like(x), torch.empty_like(x)
        else:
            w0, w1 = d.workspace(x)
        ev[0].record()
        d.exchange(x, w0); ev[1].record()
        d.stages.butterfly(w0, w1, direction); ev[2].record()
        d.exchange(w1, w0); ev[3].record()
        d.stages.local(w0, out if cyclic else w1, direction); ev[4].record()
        if cyclic:
            ev[5].record(); ev[6].record()
        else:
            d.exchange(w1, w0); ev[5].record()
            d.stages.unpack(w0, out); ev[6].record()
    torch.cuda.synchronize(dev)
    stages = torch.tensor([ev[i].elapsed_time(ev[i + 1]) for i in range(6)], device=dev, dtype=torch.float64)
    dist.all_reduce(stages, op=dist.ReduceOp.MAX)
    probe = a2a_probe(m, dev, world)
    # e2e: the rank's block from pinned host memory in, the result back out, every step
    h_in = x.cpu().pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    d_in = x if a.transport == "p2p" else torch.empty_like(x)
    e2e_steps = max(1, a.e2e_steps)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        d_in.copy_(h_in, non_blocking=True)
        d.execute(d_in, direction, out=out)
        h_out.copy_(out, non_blocking=True)
        torch.cuda.synchronize(dev)
    el = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device=dev, dtype=torch.float64)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except Exception:
            pass
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        st = {k: round(float(v), 4) for k, v in zip(names, stages)}
        xms = sum(v for k, v in st.items() if "exchange" in k)
        wire = (2 if cyclic else 3) * 8 * m * (world - 1) / world
        local_plan = d.stages.describe_local().splitlines()
        print(json.dumps({
            "metric": METRIC, "value": round(gflop(n, 1) / (ms / 1e3), 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: the reference's seeded_input(N, 1) (verify.cpp:55-78) generated on the device, "
                    "block-distributed", "impl": "ours",
            "config": {"workload": f"single c2c fp32 FFT N={n} block-distributed over {world} GPU(s): "
                                   + ("P-point butterfly + local N/P plan, cyclic output order, 2 contiguous all-to-alls "
                                      if cyclic else
                                      "P-point butterfly + local N/P plan + unpack, 3 contiguous all-to-alls ")
                                   + f"({'fused into the kernels over symmetric memory' if a.transport == 'p2p' else 'NCCL'})",
                       "transport": a.transport, "output_order": a.order,
                       "n": n, "block_per_gpu": m, "chunk": m // world, "direction": a.direction,
                       "l2": "blocks of 8N/P bytes exceed the 126 MB L2 for N >= 2^25; no flush"},
            "stages_ms": st,
            "roofline": ({"bound": "nvlink", "achieved": round(wire / (xms / 1e3) / 1e9, 1) if xms else None,
                          "peak": round(probe["gbs"], 1), "unit": "GB/s",
                          "frac": round(wire / (xms / 1e3) / 1e9 / probe["gbs"], 4) if xms else None,
                          "peak_source": "measured all_to_all_single probe in this run", "traffic": None}
                         if world > 1 else
                         {"bound": "hbm", "achieved": round(16.0 * n / (ms / 1e3) / 1e9, 1), "peak": hbm,
                          "unit": "GB/s", "frac": round(16.0 * n / (ms / 1e3) / 1e9 / hbm, 4), "traffic": None,
                          "note": "single-pass 16N fraction; one rank does butterfly + local passes + unpack + "
                                  "3 device-copy exchanges"}),
            "a2a_probe": probe,
            "local_plan": local_plan[2:] if len(local_plan) > 2 else local_plan,
            "e2e": {"value": round(gflop(n, 1) / float(el[0]), 2), "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 8 * m,
                    "ms_per_step": round(float(el[0]) * 1e3, 3), "path": "DistributedFFT.execute with pinned "
                    "host block copies in and out per rank"},
            "gpu_launches": a.steps * ((1 if cyclic else 2) + d.stages.local_launches()),
            "clocks": clk.summary()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    a = parse()
    if relaunch_if_needed(a):
        return
    if a.launch_selftest:
        launch_selftest(a)
    elif a.impl == "reference":
        run_reference(a)
    elif a.workload == "distributed":
        run_distributed(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
