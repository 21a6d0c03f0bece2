"""CPU: pin the C restatement (oracle/fftgen_oracle.c) to the reference.

Every comparison here is against golden vectors produced by the UNMODIFIED
reference (tests/golden/make_golden.py) or, where oracle/_ref exists, against
the reference library itself.  Bit-exact unless stated: the restatement
follows the lowered arithmetic of lower_complex.cpp operation for operation.
"""
import os

import numpy as np
import pytest

import oracle


def test_seeded_input_matches_reference(orc, golden):
    # verify.cpp:69-78; SURVEY Appendix A pins seeded_input(4,1) and (1,0)
    for key in golden.files:
        if key.startswith("seeded_"):
            _, n, seed = key.split("_")
            assert np.array_equal(orc.seeded_input(int(n), int(seed)), golden[key]), key
    x = orc.seeded_input(4, 1)
    assert x[0] == float.fromhex("0x1.10a2dec890258p-3")
    assert x[1] == float.fromhex("0x1.f75c6d0b2c774p-2")
    assert x[6] == float.fromhex("0x1.8267b1b35cd8ep-1")
    assert orc.seeded_input(1, 0)[0] == 0.76662161642728521


def test_seeded_input_deterministic_and_in_range(orc):
    a, b, c = orc.seeded_input(32, 99), orc.seeded_input(32, 99), orc.seeded_input(32, 100)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert (a >= -1.0).all() and (a < 1.0).all()


def test_unit_root_matches_reference(orc, golden):
    # matrix.cpp:14-35, exact quadrants
    for n in (1, 2, 4, 8, 16, 64, 1024):
        want = golden[f"unit_root_{n}"]
        got = np.array([[orc.unit_root(n, t).real, orc.unit_root(n, t).imag] for t in range(n)])
        assert np.array_equal(got, want), n
    assert orc.unit_root(4, 1) == complex(0.0, -1.0)
    assert orc.unit_root(8, 6) == complex(0.0, 1.0)


def test_pipeline_text_matches_reference(orc, golden_meta):
    # print_pipeline goldens (rewrite.cpp:275-296) for both planners
    for key, text in golden_meta["pipelines"].items():
        alg, n, radix = key.rsplit("_", 2)
        assert orc.pipeline_text(int(n), alg, int(radix)) == text, key


def test_pipeline_golden_text_test_rewrite():
    # test_rewrite.cpp:194-201
    o = oracle.Oracle()
    assert o.pipeline_text(4, "cooley-tukey", 2) == (
        "Permute(m=2, total=4)\nFusedIKMV(n=2, copies=2)\nTwiddleMul(len=4)\nFusedMKIV(m=2, copies=2)\n")


def test_index_maps_and_twiddle_exponents_match_reference(orc, golden, golden_meta):
    # bit-exact plan/permutation indices, exponents of w_s
    checked = 0
    for key, nops in golden_meta["num_ops"].items():
        alg, n, radix = key.rsplit("_", 2)
        n, radix = int(n), int(radix)
        ops = orc.fuse(n, alg, radix)
        assert len(ops) == nops, key
        for i, op in enumerate(ops):
            if f"map_{key}_{i}" in golden.files:
                assert np.array_equal(orc.op_index_map(op, n), golden[f"map_{key}_{i}"]), (key, i)
                checked += 1
            if f"tw_{key}_{i}" in golden.files:
                exps, s = golden[f"tw_{key}_{i}"]
                assert op.tw_total == s[0], (key, i)
                assert np.array_equal(orc.op_twiddle_exps(op, n), exps), (key, i)
                checked += 1
    assert checked > 200


def test_appendix_a_goldens(orc):
    ops = orc.fuse(16, "stockham", 4)
    perm = [op for op in ops if op.kind == 4][0]
    assert list(orc.op_index_map(perm, 16)) == [0, 4, 8, 12, 1, 5, 9, 13, 2, 6, 10, 14, 3, 7, 11, 15]
    twd = [op for op in ops if op.kind == 3][0]
    assert list(orc.op_twiddle_exps(twd, 16)) == [0, 0, 0, 0, 0, 1, 2, 3, 0, 2, 4, 6, 0, 3, 6, 9]
    assert orc.stockham_radices(1024, 8) == [2, 8, 8, 8]
    assert orc.stockham_radices(32, 4) == [2, 4, 4]


@pytest.mark.parametrize("alg,radix", [("cooley-tukey", 2), ("stockham", 4), ("stockham", 8),
                                       ("stockham", 2)])
def test_forward_bit_exact_vs_reference_goldens(orc, golden, alg, radix):
    for n in (2, 4, 8, 16, 64, 256, 1024, 4096):
        x = orc.seeded_input(n, 1)
        got = orc.forward(x, alg, radix)
        assert np.array_equal(got, golden[f"fwd_{alg}_{radix}_{n}_1"]), (alg, radix, n)


def test_gpu_goldens_reproduced(orc, golden, golden_meta):
    for n, seed in golden_meta["gpu_goldens"]:
        x = golden[f"gpu_in_{n}_{seed}"].astype(np.float64)
        assert np.array_equal(orc.forward(x, "stockham", 4), golden[f"gpu_out_{n}_{seed}"])


def test_known_answers(orc, golden):
    # test_exec.cpp:81-99: delta -> ones; DFT_2(1,2) = (3,-1) exactly
    delta = np.zeros(8)
    delta[0] = 1.0
    assert np.array_equal(orc.forward(delta, "cooley-tukey", 2), golden["kat_delta4_out"])
    assert np.array_equal(orc.forward(np.array([1.0, 0, 2.0, 0]), "cooley-tukey", 2), [3.0, 0.0, -1.0, 0.0])
    # dft_oracle restatement (verify.cpp:19-37), bit-exact
    assert np.array_equal(orc.dft_oracle(orc.seeded_input(8, 77)), golden["dft_oracle_8_77"])
    assert np.array_equal(orc.dft_oracle(orc.seeded_input(64, 17)), golden["dft_oracle_64_17"])


def test_oracle_properties(orc):
    # Parseval and linearity (test_verify.cpp:29-59), inverse round trip
    x = orc.seeded_input(64, 17)
    X = orc.dft_oracle(x)
    assert abs((X ** 2).sum() - 64 * (x ** 2).sum()) / (64 * (x ** 2).sum()) < 1e-9
    for n in (8, 64, 512):
        a, b = orc.seeded_input(n, 5), orc.seeded_input(n, 6)
        za, zb = oracle.as_complex(a), oracle.as_complex(b)
        mix = oracle.as_interleaved(0.7 * za + 1.1j * zb)
        lhs = oracle.as_complex(orc.forward(mix, "stockham", 4))
        rhs = 0.7 * oracle.as_complex(orc.forward(a, "stockham", 4)) + 1.1j * oracle.as_complex(
            orc.forward(b, "stockham", 4))
        assert np.abs(lhs - rhs).max() / np.abs(rhs).max() < 1e-12
        back = orc.forward(orc.forward(a, "stockham", 4), "stockham", 4, inverse=True) / n
        assert np.abs(back - a).max() < 1e-13


def test_sampled_bins_match_full_oracle(orc):
    n = 4096
    x = orc.seeded_input(n, 3)
    full = orc.forward(x, "stockham", 4)
    bins = [0, 1, 7, 1000, 2048, 4095]
    got = orc.dft_bins(x, bins)
    want = np.concatenate([full[2 * b:2 * b + 2] for b in bins])
    assert np.abs(got - want).max() < 1e-9
    inv = orc.dft_bins(x, bins, inverse=True)
    full_inv = orc.forward(x, "stockham", 4, inverse=True)
    assert np.abs(inv - np.concatenate([full_inv[2 * b:2 * b + 2] for b in bins])).max() < 1e-9


def test_error_metric_and_mflops(orc, golden_meta):
    a = np.array([1, 1, 2, 2, 3, 3, 4, 4], dtype=np.float64)
    b = a.copy()
    b[4] += 4e-7
    assert orc.error_metric(a, a) == 0.0
    assert abs(orc.error_metric(a, b) - 1e-7) < 1e-12  # doctest Approx(1e-7).epsilon(1e-12)
    for key, want in golden_meta["mflops"].items():
        n, s = key.split("_")
        assert orc.mflops(int(n), float(s)) == want


def test_oracle_matches_live_reference(orc, ref):
    """Direct cross-check against the reference library when it is built."""
    for n in (1, 2, 8, 32, 512, 2048):
        for alg, radix in (("cooley-tukey", 2), ("cooley-tukey", 4), ("stockham", 16)):
            x = orc.seeded_input(n, 9)
            assert np.array_equal(orc.forward(x, alg, radix), ref.forward(x, alg, radix)), (n, alg, radix)
    x = orc.seeded_input(256, 4)
    split = ref.forward(oracle.relayout_to_split(x), "stockham", 4, "split")
    assert np.array_equal(oracle.split_to_interleaved(split), orc.forward(x, "stockham", 4))


def test_plan_errors_mirror_reference(orc):
    with pytest.raises(RuntimeError):
        orc.fuse(12, "stockham", 4)   # PlanError: not a power of two
    with pytest.raises(RuntimeError):
        orc.fuse(16, "stockham", 3)   # PlanError: radix not a power of two
    with pytest.raises(RuntimeError):
        orc.fuse(256, "stockham", 128)  # FuseError: kernel cap 64


def test_reference_aot_path_matches_interpreter(ref):
    """The reference's emit_c output (oracle/_ref/libref_aot.so, the CPU
    baseline's ahead-of-time leg) is bitwise the reference interpreter."""
    if not os.path.exists(oracle.AOT_SO):
        pytest.skip("oracle/_ref/libref_aot.so not built (reference tree absent)")
    a = oracle.AotRef()
    x = oracle.relayout_to_split(np.stack([ref.seeded_input(a.N, 1 + b) for b in range(6)]))
    got = a.forward(x, threads=3)
    want = ref.forward(x, a.ALG, a.RADIX, a.LAYOUT, threads=3)
    assert np.array_equal(got, want)
