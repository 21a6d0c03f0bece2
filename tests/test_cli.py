"""The fftgen-b200 CLI (paper_2308_00497_b200/tools/fftgen_cli.cpp), restating
the reference's CLI integration tests (proj/tests/test_cli.cpp)."""
import csv
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2308_00497_b200", "lib", "fftgen-b200")


def run(*args, timeout=600):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)


def test_usage_errors_exit_2():
    # test_cli.cpp:92-101
    assert run().returncode == 2
    assert run("bogus").returncode == 2
    assert run("verify", "--sizes", "12,16").returncode == 2
    assert run("compile", "--size", "16", "--layout", "diagonal", "--emit", "ir").returncode == 2


def test_plan_errors_exit_1():
    # shape errors are usage errors at the CLI (StageFlags::to_config, main.cpp:62-72);
    # what the planner / lowering reject exits 1 with the reference's class
    assert run("compile", "--size", "12", "--emit", "ir").returncode == 2
    p = run("compile", "--size", "256", "--algorithm", "stockham", "--radix", "128", "--emit", "ir")
    assert p.returncode == 1 and "FuseError" in p.stderr
    p = run("compile", "--size", "64", "--vectorize", "inner", "--vector-width", "6", "--emit", "ir")
    assert p.returncode == 1 and "LowerError" in p.stderr


def test_compile_emit_formula_and_ir_goldens(golden_meta):
    """--emit formula / ir are host-only and byte-identical to the reference's
    print_formula / print_pipeline (formula.cpp:104-146, rewrite.cpp:275-296)
    for every golden configuration (tests/golden, generated from oracle/_ref)."""
    for key, text in golden_meta["formulas"].items():
        alg, n, r = key.rsplit("_", 2)
        p = run("compile", "--size", n, "--algorithm", alg, "--radix", r, "--emit", "formula")
        assert p.returncode == 0 and p.stdout == text + "\n", key
    for key, text in golden_meta["pipelines"].items():
        alg, n, r = key.rsplit("_", 2)
        p = run("compile", "--size", n, "--algorithm", alg, "--radix", r, "--emit", "ir")
        assert p.returncode == 0 and p.stdout == text, key


def test_emit_outputs_byte_stable_without_gpu():
    # test_cli.cpp:76-89 / acceptance.cpp:350-368 for the host-only texts
    for emit in ("formula", "ir", "loops"):
        args = ("compile", "--size", "64", "--algorithm", "stockham", "--radix", "4", "--vectorize", "inner",
                "--interleaved-opt", "--emit", emit)
        a, b = run(*args), run(*args)
        assert a.returncode == 0 and a.stdout and a.stdout == b.stdout, emit
    # 2^24: two 4096-point groups interleaved, three 256-point groups split (measured defaults)
    loops = run("compile", "--size", str(1 << 24), "--emit", "loops").stdout
    assert loops.startswith("four-step: 2 group launches") and "HBM scratch -> HBM" in loops
    loops = run("compile", "--size", str(1 << 24), "--layout", "split", "--emit", "loops").stdout
    assert loops.startswith("four-step: 3 group launches") and "HBM scratch -> HBM" in loops
    c = run("compile", "--size", "16", "--emit", "c")
    assert c.returncode == 1 and "LowerError" in c.stderr


@pytest.mark.gpu
def test_compile_emit_ir_golden(golden_meta):
    # the reference's own print_pipeline text (test_rewrite.cpp:194-201, test_cli.cpp:44-48)
    p = run("compile", "--size", "4", "--emit", "ir")
    assert p.returncode == 0
    assert p.stdout == golden_meta["pipelines"]["cooley-tukey_4_2"]
    p = run("compile", "--size", "4096", "--algorithm", "stockham", "--radix", "8", "--emit", "radices")
    assert p.stdout.split() == ["8", "8", "8", "8"]
    assert "fft_block_tma_kernel<4096>" in run("compile", "--size", "4096", "--emit", "kernels").stdout


@pytest.mark.gpu
def test_run_size1_is_seeded_identity():
    # test_cli.cpp:50-58: N=1 with --random 0 prints seeded_input(1, 0) (fp32-rounded on this path)
    p = run("run", "--size", "1", "--random", "0")
    re, im = (float(v) for v in p.stdout.split())
    assert abs(re - 0.76662161642728521) < 1e-7 and abs(im + 0.13694400590298006) < 1e-7


@pytest.mark.gpu
def test_verify_matrix_passes():
    # verify.cpp:127-181 with the reference gate 1e-7
    p = run("verify", "--sizes", "16..4096", "--inputs", "3")
    assert p.returncode == 0, p.stdout[-2000:]
    lines = p.stdout.splitlines()
    assert lines[-1].endswith(", 0 failed")
    assert all(l.startswith("PASS ") for l in lines[:-1])
    # both algorithms x radices {2,4,16} x (5 vector modes interleaved + 3 split), verify.cpp:136-155
    assert len(lines) - 1 == sum(2 * len([r for r in (2, 4, 16) if r <= n]) * 8 for n in [16 << i for i in range(9)])


@pytest.mark.gpu
def test_bench_csv_schema(tmp_path):
    out = tmp_path / "b.csv"
    p = run("bench", "--device", "--sizes", "1024,4096", "--repeats", "5", "--batch", "64", "--csv", out)
    assert p.returncode == 0, p.stderr
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0])[:9] == ["n", "algorithm", "radix", "layout", "vector_mode", "repeats", "mean_seconds",
                                 "mflops", "seed"]
    for r in rows:
        assert float(r["mean_seconds"]) > 0 and float(r["gflops"]) > 0
        assert abs(float(r["mflops"]) / 1e3 - float(r["gflops"])) / float(r["gflops"]) < 1e-3


# ---- the reference's own tests/test_cli.cpp, compiled unchanged (oracle/Makefile)
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "ref_test_cli")


def ref_cli_test():
    if not os.path.exists(REF_CLI):
        if os.path.exists("/root/reference/proj/tests/test_cli.cpp"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, stdout=subprocess.DEVNULL)
        else:
            pytest.skip("oracle/_ref/ref_test_cli not built")
    if not os.path.exists("/root/repo/paper_2308_00497_b200/lib/fftgen-b200"):
        pytest.skip("the compiled-in CLI path /root/repo/... is absent")
    return REF_CLI


def test_reference_test_cli_host_cases():
    p = subprocess.run([ref_cli_test(), "-tc=compile --emit formula*,usage errors*"], capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0 and "2 passed, 0 failed" in p.stdout, p.stdout + p.stderr


@pytest.mark.gpu
def test_reference_test_cli_all_cases():
    """All seven cases of the reference's test_cli.cpp against fftgen-b200: formula
    text, run --size 1 identity, input files, byte-stable emits, usage exit
    codes, the verify sweep and the bench CSV schema."""
    p = subprocess.run([ref_cli_test()], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and "7 passed, 0 failed" in p.stdout, p.stdout + p.stderr
