"""CPU: the product's host plan builder and C ABI surface (no GPU needed).

* the library loads and exports every symbol include/fftgen_b200.h declares,
* plan introspection (radices, fused op list, index maps, twiddle exponents,
  print_pipeline text) is bit-exact against the reference's goldens,
* the compile-time butterfly constants equal unit_root rounded to fp32,
* the pass regrouping the kernels execute is restated in numpy and matches
  the oracle,
* the error behaviour at plan creation mirrors the reference's exceptions.
Plan creation needs a CUDA device, so these tests exercise the host builder
through a C++ test driver linked to the same objects (tests/cpp/).
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "fftgen_b200.h")
LIB = os.path.join(ROOT, "paper_2308_00497_b200", "lib", "libfftgen_b200.so")
CSRC = os.path.join(ROOT, "paper_2308_00497_b200", "csrc")
PLAN_TOOL = os.path.join(ROOT, "paper_2308_00497_b200", "build", "plan_tool")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(
        r"^(?:fftgen_status|int|int64_t|void|size_t|const char \*|const fftgen_plan \*)\s*\*?(fftgen_[a-z0-9_]+)\(",
        text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    import paper_2308_00497_b200 as fg
    assert set(fg.ABI_SYMBOLS) == set(syms)
    assert lib.fftgen_abi_version() == 3


def test_error_strings_and_config_defaults():
    import paper_2308_00497_b200 as fg
    lib = fg.lib
    assert lib.fftgen_error_string(1) == b"PlanError"
    assert lib.fftgen_error_string(2) == b"DimensionError"
    assert lib.fftgen_error_string(3) == b"ExecError"
    c = fg._Config()
    lib.fftgen_config_init(ctypes.byref(c))
    # PipelineConfig defaults (driver.hpp:26-35): Cooley-Tukey, radix 2, interleaved
    assert (c.algorithm, c.radix, c.layout, c.batch, c.device) == (0, 2, 0, 1, 0)
    # vec None, vector_width 8, interleaved_opt off, no tile; measured-default kernels
    assert (c.vec, c.vector_width, c.interleaved_opt, c.tile_kind) == (0, 8, 0, 0)
    assert (c.tuning, c.cluster_size, c.host_chunk_mb) == (0, 0, 0)
    assert ctypes.sizeof(c) == 72
    for code, name in ((8, b"LowerError"), (9, b"BoundsError"), (10, b"GpuMapError")):
        assert lib.fftgen_error_string(code) == name


@pytest.mark.parametrize("kw,msg", [
    (dict(vec="inner", vector_width=6), "power of two"),
    (dict(vec="outer", vector_width=128), "capped at 64"),
    (dict(tile=("exact", 0)), "must be positive"),
    (dict(tile=("cache", -5)), "must be positive"),
])
def test_schedule_options_rejected_like_vectorize_and_tile(kw, msg):
    """PipelineConfig.vec / vector_width / tile are validated the way the
    reference's vectorize() and tile() validate them (transforms.cpp:85-95,
    349-354): LowerError, raised before any device is touched."""
    import paper_2308_00497_b200 as fg
    with pytest.raises(fg.LowerError, match=msg):
        fg.compile_pipeline(fg.PipelineConfig(n=64, **kw))


@pytest.fixture(scope="module")
def plan_tool():
    """C++ driver over the host plan builder (plan.cpp), no CUDA device needed."""
    src = os.path.join(ROOT, "tests", "cpp", "plan_tool.cpp")
    if (not os.path.exists(PLAN_TOOL)) or os.path.getmtime(PLAN_TOOL) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(CSRC, "plan.cpp"))):
        os.makedirs(os.path.dirname(PLAN_TOOL), exist_ok=True)
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", CSRC, "-o", PLAN_TOOL, src,
                        os.path.join(CSRC, "plan.cpp"), os.path.join(CSRC, "geom.cpp")], check=True)
    def run(*args):
        p = subprocess.run([PLAN_TOOL, *map(str, args)], capture_output=True, text=True)
        return p.returncode, p.stdout, p.stderr
    return run


def test_pipeline_text_matches_reference_goldens(plan_tool, golden_meta):
    for key, text in golden_meta["pipelines"].items():
        alg, n, radix = key.rsplit("_", 2)
        rc, out, err = plan_tool("text", n, 0 if alg == "cooley-tukey" else 1, radix)
        assert rc == 0, err
        assert out == text, key


def test_index_maps_bit_exact_vs_reference(plan_tool, golden, golden_meta):
    checked = 0
    for key in golden_meta["num_ops"]:
        alg, n, radix = key.rsplit("_", 2)
        a = 0 if alg == "cooley-tukey" else 1
        rc, out, err = plan_tool("maps", n, a, radix)
        assert rc == 0, err
        for line in out.splitlines():
            idx, kind, s, *vals = line.split()
            vals = np.array([int(v) for v in vals])
            if kind in ("2", "4"):
                assert np.array_equal(vals, golden[f"map_{key}_{idx}"]), (key, idx)
                checked += 1
            elif kind == "3":
                exps, ss = golden[f"tw_{key}_{idx}"]
                assert int(s) == ss[0] and np.array_equal(vals, exps), (key, idx)
                checked += 1
    assert checked > 200


def test_radices_reference_order(plan_tool):
    for n, r, want in ((1024, 8, [2, 8, 8, 8]), (32, 4, [2, 4, 4]), (4096, 4, [4] * 6),
                       (2048, 8, [4, 8, 8, 8]), (1, 2, [])):
        rc, out, _ = plan_tool("radices", n, r)
        assert rc == 0
        assert [int(v) for v in out.split()] == want


def test_plan_errors(plan_tool):
    # formula.cpp:150-160 / rewrite.cpp:56-62 behaviour: PlanError / FuseError
    assert plan_tool("text", 12, 1, 4)[0] == 1
    assert plan_tool("text", 16, 1, 3)[0] == 1
    assert plan_tool("text", 16, 1, 1)[0] == 1
    assert plan_tool("text", 256, 1, 128)[0] == 4
    assert plan_tool("text", 64, 1, 128)[0] == 0   # r = min(radix, n) = 64 fits the cap


def test_exec_plan_passes_cover_all_sizes(plan_tool):
    for l2 in range(0, 15):
        rc, out, err = plan_tool("passes", 1 << l2)
        assert rc == 0, err
        passes = [tuple(int(v) for v in ln.split()) for ln in out.splitlines()]
        prod = 1
        for R, cols, k, s in passes:
            assert cols == prod and s == R * cols and k * s == (1 << l2)
            prod *= R
        assert prod == 1 << l2


def test_pass_radix_hint_steers_block_passes(plan_tool):
    """fftgen_config.pass_radix (the radix hint): register passes of at most
    that radix in the reference's Stockham shape, remainder radix first
    (formula.cpp:182-195), where <= 3 passes suffice and the default differs;
    otherwise the default plan."""
    def passes(n, hint=0, layout=0):
        rc, out, err = plan_tool("passes", n, hint, layout)
        assert rc == 0, err
        return [int(ln.split()[0]) for ln in out.splitlines()]
    assert passes(4096) == [64, 64]
    # measured defaults: radix-8 three-pass plans at 2^7..2^9; 64 keeps the two-pass ones
    assert passes(256) == [4, 8, 8] and passes(512) == [8, 8, 8] and passes(128) == [2, 8, 8]
    # interleaved 2^10 / 2^11: radix-16 three-pass (direct kernel); split keeps two passes
    assert passes(1024) == [4, 16, 16] and passes(2048) == [8, 16, 16]
    assert passes(1024, 0, 1) == [32, 32] and passes(2048, 0, 1) == [32, 64] and passes(2048, 64) == [32, 64]
    assert passes(256, 64) == [16, 16] and passes(512, 64) == [16, 32] and passes(128, 64) == [8, 16]
    assert passes(4096, 16) == [16, 16, 16] and passes(4096, 32) == [4, 32, 32]
    assert passes(2048, 16) == [8, 16, 16] and passes(2048, 32) == [2, 32, 32]
    assert passes(1024, 16) == [4, 16, 16] and passes(512, 16) == [2, 16, 16]
    assert passes(512, 8) == [8, 8, 8] and passes(256, 8) == [4, 8, 8] and passes(128, 8) == [2, 8, 8]
    assert passes(1024, 8) == [2, 8, 8, 8] and passes(2048, 8) == [4, 8, 8, 8]
    assert passes(256, 16) == passes(256, 64)                                            # the default fits
    assert passes(1 << 13, 16) == [2, 16, 16, 16] and passes(1 << 14, 16) == [4, 16, 16, 16]
    assert passes(4096, 8) == [8, 8, 8, 8] and passes(1 << 13, 8) == passes(1 << 13)    # > 4 passes: default
    assert passes(1 << 14, 32) == passes(1 << 14) and passes(64, 64) == passes(64)
    assert plan_tool("passes", 4096, 12)[0] == 1                                        # PlanError
    for n in (128, 256, 512, 1024, 2048, 4096):
        for hint in (8, 16, 32):
            rs = passes(n, hint)
            prod = 1
            for r in rs:
                prod *= r
            assert prod == n and len(rs) <= 4


def test_fourstep_group_splits_follow_the_measured_table(plan_tool):
    """group_split (plan.cpp): the per-size, per-layout splits chosen from the
    measured per-launch rates."""
    def ns(n, layout):
        rc, out, err = plan_tool("passes", n, 0, layout)
        assert rc == 0, err
        return [int(ln.split()[0]).bit_length() - 1 for ln in out.splitlines()]
    il, sp = 0, 1
    assert ns(1 << 16, il) == [8, 8] and ns(1 << 17, sp) == [9, 8]
    assert ns(1 << 18, il) == [10, 8] and ns(1 << 18, sp) == [10, 8]
    assert ns(1 << 19, il) == [11, 8] and ns(1 << 19, sp) == [10, 9]
    assert ns(1 << 20, il) == [12, 8] and ns(1 << 20, sp) == [10, 10]
    assert ns(1 << 21, il) == [11, 10] and ns(1 << 21, sp) == [10, 11]
    assert ns(1 << 23, il) == [11, 12] and ns(1 << 23, sp) == [12, 11]
    assert ns(1 << 24, il) == [12, 12] and ns(1 << 24, sp) == [8, 8, 8]
    assert ns(1 << 26, il) == [8, 8, 10] and ns(1 << 28, sp) == [8, 9, 11]
    assert ns(1 << 29, il) == [8, 9, 12] and len(ns(1 << 29, sp)) == 4
    assert ns(1 << 30, il) == [8, 11, 11] and len(ns(1 << 30, sp)) == 4


def test_fourstep_groups_cover_large_sizes(plan_tool):
    """K3 groups: each a radix-NS Stockham stage with cols = prior product,
    k = N / s; inner groups need k >= tile, the last group has k == 1."""
    for l2 in range(15, 31):
        rc, out, err = plan_tool("passes", 1 << l2)
        assert rc == 0, err
        groups = [tuple(int(v) for v in ln.split()) for ln in out.splitlines()]
        assert 2 <= len(groups) <= 4
        prod = 1
        for R, cols, k, s in groups:
            assert 64 <= R <= 4096 and cols == prod and s == R * cols and k * s == 1 << l2
            prod *= R
        assert prod == 1 << l2 and groups[-1][2] == 1
    assert plan_tool("passes", 1 << 31)[0] == 1  # PlanError above 2^30


def test_fourstep_regrouping_restated_matches_oracle(plan_tool, orc):
    for n in (1 << 15, 1 << 16):
        rc, out, _ = plan_tool("passes", n)
        groups = [tuple(int(v) for v in ln.split()) for ln in out.splitlines()]
        x = orc.seeded_input(n, 3)
        z = oracle.as_complex(x)
        for R, cols, k, s in groups:
            # vectorised radix-R Stockham stage over the whole transform
            m = np.arange(cols)[:, None, None]
            A = np.arange(R)[None, :, None]
            c = np.arange(k)[None, None, :]
            v = z[(m * R + A) * k + c] * np.exp(-2j * np.pi * A * m / s)
            V = np.fft.fft(v, axis=1)
            y = np.empty_like(z)
            y[(A * cols + m) * k + c] = V
            z = y
        want = oracle.as_complex(orc.forward(x, "stockham", 4))
        assert np.abs(z - want).max() / np.abs(want).max() < 1e-12


def test_butterfly_constants_are_unit_root_fp32(orc):
    text = open(os.path.join(CSRC, "roots64.cuh")).read()
    def arr(name):
        body = text.split(name + "[64] = {")[1].split("}")[0]
        return [float.fromhex(v.strip().rstrip("f")) if "0x" in v else float(v.strip().rstrip("f"))
                for v in body.split(",")]
    re_, im_ = arr("kRoot64Re"), arr("kRoot64Im")
    for j in range(64):
        w = orc.unit_root(64, j)
        assert np.float32(w.real) == np.float32(re_[j]) and np.float32(w.imag) == np.float32(im_[j]), j


def _pass(x, R, cols, n, sign=-1):
    s = cols * R
    k = n // s
    y = np.empty_like(x)
    A = np.arange(R)
    for m in range(cols):
        for c in range(k):
            v = x[(m * R + A) * k + c] * np.exp(sign * 2j * np.pi * A * m / s)
            V = np.fft.fft(v) if sign < 0 else np.fft.ifft(v) * R
            y[(A * cols + m) * k + c] = V
    return y


def test_pass_regrouping_restated_matches_oracle(plan_tool, orc):
    """The kernels' pass formula (fft_block.cuh header) restated in numpy."""
    for n in (16, 128, 1024, 2048, 8192):
        rc, out, _ = plan_tool("passes", n)
        passes = [tuple(int(v) for v in ln.split()) for ln in out.splitlines()]
        x = orc.seeded_input(n, 2)
        z = oracle.as_complex(x)
        for R, cols, k, s in passes:
            z = _pass(z, R, cols, n)
        want = oracle.as_complex(orc.forward(x, "stockham", 2))
        assert np.abs(z - want).max() / np.abs(want).max() < 1e-12, n


def test_block_twiddle_tables_bit_exact(plan_tool, orc):
    # fp32 tables = unit_root(s, A*m) rounded once (formula.cpp:199-206 values)
    rc, out, _ = plan_tool("twiddles", 4096)
    vals = np.array([float.fromhex(v) for v in out.split()], dtype=np.float64)
    assert vals.size == 2 * 64 * 64
    want = []
    for A in range(64):
        for m in range(64):
            w = orc.unit_root(4096, A * m)
            want += [w.real, w.imag]
    assert np.array_equal(vals.astype(np.float32), np.array(want).astype(np.float32))
