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
    p = run("compile", "--size", "12", "--emit", "ir")
    assert p.returncode == 1 and "PlanError" in p.stderr


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
    assert len(lines) - 1 == sum(2 * len([r for r in (2, 4, 16) if r <= n]) * 2 for n in [16 << i for i in range(9)])


@pytest.mark.gpu
def test_bench_csv_schema(tmp_path):
    out = tmp_path / "b.csv"
    p = run("bench", "--sizes", "1024,4096", "--repeats", "5", "--batch", "64", "--csv", out)
    assert p.returncode == 0, p.stderr
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0])[:9] == ["n", "algorithm", "radix", "layout", "vector_mode", "repeats", "mean_seconds",
                                 "mflops", "seed"]
    for r in rows:
        assert float(r["mean_seconds"]) > 0 and float(r["gflops"]) > 0
        assert abs(float(r["mflops"]) / 1e3 - float(r["gflops"])) / float(r["gflops"]) < 1e-3
