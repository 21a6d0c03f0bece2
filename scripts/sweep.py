#!/usr/bin/env python
"""Size / layout / variant sweep in one process (development tool, not the bench).

    python scripts/sweep.py --sizes 14,15,16 --layouts split,interleaved \
        --variants default,cluster_size=-1 [--bytes 1073741824] [--inverse]

Per row: CUDA-event time of `steps` back-to-back executes on device-resident
inputs of ~`bytes` per GPU (inputs + outputs far larger than L2), GFLOP/s of
5 N log2 N and the fraction of the measured HBM peak for 16 N bytes per
transform.  Variant = PipelineConfig field overrides KEY=INT joined by '+'
(tuning=<FFTGEN_TUNE_* bits>, cluster_size=C).
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="10,11,12,13,14,15,16")
    ap.add_argument("--layouts", default="split,interleaved")
    ap.add_argument("--variants", default="default")
    ap.add_argument("--bytes", type=int, default=1 << 30, help="input bytes per GPU")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--inverse", action="store_true")
    ap.add_argument("--batch", type=int, default=0, help="override batch")
    a = ap.parse_args()

    import torch
    import paper_2308_00497_b200 as fg

    peak = 6549.1
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    direction = fg.INVERSE if a.inverse else fg.FORWARD
    for l2 in [int(s) for s in a.sizes.split(",")]:
        n = 1 << l2
        batch = a.batch or max(1, a.bytes // (8 * n))
        for layout in a.layouts.split(","):
            if layout == "split":
                in0 = torch.rand(batch, n, device="cuda") * 2 - 1
                in1 = torch.rand(batch, n, device="cuda") * 2 - 1
                out0, out1 = torch.empty_like(in0), torch.empty_like(in1)
            else:
                in0 = torch.rand(batch, n, 2, device="cuda") * 2 - 1
                in1 = out1 = None
                out0 = torch.empty_like(in0)
            ref = None
            for var in a.variants.split(","):
                kw = {}
                if var != "default":
                    for kv in var.split("+"):
                        k, v = kv.split("=", 1)
                        kw[k] = int(v, 0)
                plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, **kw))
                for _ in range(a.warmup):
                    plan.execute(in0, out0, in1, out1, direction=direction)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(a.steps):
                    plan.execute(in0, out0, in1, out1, direction=direction)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e) / a.steps
                tf = 5 * n * l2 * batch / (ms / 1e3) / 1e12
                frac = 16 * n * batch / (ms / 1e3) / 1e9 / peak
                same = None
                if ref is None:
                    ref = out0.clone()
                else:
                    same = bool(torch.equal(ref, out0))
                kern = next((w for w in plan.describe().split() if "kernel<" in w), "?")
                print(json.dumps({"n": f"2^{l2}", "layout": layout, "variant": var, "batch": batch,
                                  "ms": round(ms, 4), "TFLOPs": round(tf, 2), "frac": round(frac, 3),
                                  "launches": plan.launches(), "kernel": kern, "bitwise_eq_first": same}),
                      flush=True)
                plan.close()
            del in0, in1, out0, out1, ref
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
