"""Generate tests/golden/golden.npz + golden.json from the UNMODIFIED reference.

Run in the build container (where /root/reference exists and
oracle/_ref/libfftgen_ref.so has been built by `make -C oracle`):

    python tests/golden/make_golden.py

Every array comes from the reference's own public API through the forwarding
shim oracle/ref_shim.cpp (compile_pipeline+interpret, seeded_input,
dft_oracle, unit_root, fuse/apply_op, print_pipeline, print_formula).  The
fixtures pin the C restatement (oracle/fftgen_oracle.c) and are the GPU
parity goldens; they travel to the GPU box, /root/reference does not.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32_round(x: np.ndarray) -> np.ndarray:
    return x.astype(np.float32).astype(np.float64)


def main() -> None:
    R = oracle.Ref()
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (unmodified reference)"}

    # seeded_input KATs (verify.cpp:69-78); SURVEY Appendix A pins (4,1) and (1,0)
    for n, seed in [(1, 0), (4, 1), (8, 1), (8, 77), (64, 13), (1024, 1), (4096, 1)]:
        arrays[f"seeded_{n}_{seed}"] = R.seeded_input(n, seed)

    # unit_root (matrix.cpp:14-35) over a few sizes, all exponents
    for n in (1, 2, 4, 8, 16, 64, 1024):
        arrays[f"unit_root_{n}"] = np.array([[R.unit_root(n, t).real, R.unit_root(n, t).imag]
                                             for t in range(n)])

    # fused pipelines: text, data-movement index maps, twiddle exponents
    texts = {}
    maps = {}
    for alg in ("cooley-tukey", "stockham"):
        for n in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 4096):
            for radix in (2, 4, 8, 16):
                key = f"{alg}_{n}_{radix}"
                texts[key] = R.pipeline_text(n, alg, radix)
                if n > 1024 and alg == "cooley-tukey":
                    continue
                nops = R.num_ops(n, alg, radix)
                for i in range(nops):
                    kind = R.op_desc(n, alg, radix, i)[0]
                    if kind in (2, 4):
                        arrays[f"map_{key}_{i}"] = R.op_index_map(n, alg, radix, i)
                    elif kind == 3:
                        # total s of this twiddle: Stockham stage s / CT level n_sub;
                        # recover by trying the candidate powers of two
                        for s in [1 << b for b in range(1, 20) if (1 << b) <= n]:
                            exps, coeffs = R.op_twiddle(n, alg, radix, i, s)
                            if (exps >= 0).all():
                                arrays[f"tw_{key}_{i}"] = np.stack([exps, np.full(n, s)])
                                break
                        else:
                            raise RuntimeError(f"no exact twiddle total for {key} op {i}")
                maps[key] = nops
    meta["pipelines"] = texts
    meta["num_ops"] = maps
    meta["formulas"] = {f"{alg}_{n}_{r}": R.formula_text(n, alg, r)
                        for alg in ("cooley-tukey", "stockham") for n in (4, 8, 16, 32) for r in (2, 4)}

    # forward outputs of the reference interpreter (fp64 inputs), both algorithms
    for alg, radix in (("cooley-tukey", 2), ("stockham", 4), ("stockham", 8), ("stockham", 2)):
        for n in (2, 4, 8, 16, 64, 256, 1024, 4096):
            x = R.seeded_input(n, 1)
            arrays[f"fwd_{alg}_{radix}_{n}_1"] = R.forward(x, alg, radix)
    # KATs from test_exec.cpp / test_verify.cpp
    arrays["kat_dft2_in"] = np.array([1.0, 0.0, 2.0, 0.0])
    arrays["kat_dft2_out"] = R.forward(arrays["kat_dft2_in"], "cooley-tukey", 2)
    delta = np.zeros(8)
    delta[0] = 1.0
    arrays["kat_delta4_out"] = R.forward(delta, "cooley-tukey", 2)
    arrays["dft_oracle_8_77"] = R.dft_oracle(R.seeded_input(8, 77))
    arrays["dft_oracle_64_17"] = R.dft_oracle(R.seeded_input(64, 17))

    # GPU parity goldens: fp32-rounded seeded inputs through the reference (fp64)
    gpu = []
    for n, seeds in ((1024, (1, 2)), (4096, (1,)), (16384, (1,))):
        for seed in seeds:
            x = f32_round(R.seeded_input(n, seed))
            arrays[f"gpu_in_{n}_{seed}"] = x.astype(np.float32)
            arrays[f"gpu_out_{n}_{seed}"] = R.forward(x, "stockham", 4, "interleaved")
            gpu.append([n, seed])
    meta["gpu_goldens"] = gpu
    meta["mflops"] = {"1024_1.0": R.mflops(1024, 1.0), "2_1.0": R.mflops(2, 1.0),
                      "256_1e-6": R.mflops(256, 1e-6)}

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays")


if __name__ == "__main__":
    main()
