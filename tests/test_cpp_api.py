"""The C++ host API (include/fftgen_b200.hpp) through a compiled C++ driver
that restates the reference's exec/verify known-answer tests
(tests/cpp/api_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "api_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_2308_00497_b200", "lib")
ORCDIR = os.path.join(ROOT, "oracle")
BIN = os.path.join(ROOT, "paper_2308_00497_b200", "build", "api_test")


@pytest.fixture(scope="module")
def api_test():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", BIN, SRC,
                    "-L", LIBDIR, "-lfftgen_b200", "-L", ORCDIR, "-lfftgen_oracle",
                    f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{ORCDIR}"], check=True)
    return BIN


def test_cpp_api_host_semantics(api_test):
    p = subprocess.run([api_test, "cpu"], capture_output=True, text=True)
    assert p.returncode == 0, p.stdout + p.stderr


@pytest.mark.gpu
def test_cpp_api_known_answers_and_parity(api_test):
    p = subprocess.run([api_test, "gpu"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert " 0 failed" in p.stdout
