"""profiles/sweep_rN.jsonl -> profiles/roofline_rN.md (single-pass and
pass-aware fractions of the measured HBM peak per size, layout, direction).

    python profiles/roofline_table.py [r2]
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def passes(kernel: str, launches: int) -> int:
    if "cluster" in kernel or "block" in kernel:
        return 1
    return launches  # K3: one HBM pass per group launch


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    rows = [json.loads(l) for l in open(os.path.join(HERE, f"sweep_{tag}.jsonl"))]
    out = [f"# Roofline per configuration (round {tag[1:]}, B200, `scripts/sweep.py`)", "",
           "Single-pass fraction = 16·N·batch bytes / time / measured HBM peak (6549 GB/s);",
           "pass-aware = single-pass × HBM passes of the plan (the multi-pass bound).", "",
           "| N | layout | dir | batch | TFLOP/s | ms | kernel | passes | single-pass frac | pass-aware frac |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows:
        p = passes(d["kernel"], d["launches"])
        direction = "inv" if d["variant"] == "inverse" else "fwd"
        out.append(f"| {d['n']} | {d['layout']} | {direction} | {d['batch']} | {d['TFLOPs']} | {d['ms']} | "
                   f"`{d['kernel']}` | {p} | {d['frac']:.3f} | {min(1.5, d['frac'] * p):.3f} |")
    open(os.path.join(HERE, f"roofline_{tag}.md"), "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
