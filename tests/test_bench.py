"""bench.py's host-side contract on CPU: the rank launcher behind `--gpus N`
(torchrun re-exec, MAX/SUM reductions over gloo ranks) and the reference
arm's measured steps."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def run_bench(*args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    p = subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, timeout=timeout, env=e)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p, [json.loads(ln) for ln in lines]


@pytest.mark.parametrize("gpus", [1, 2, 4])
def test_gpus_flag_launches_that_many_ranks(gpus):
    p, lines = run_bench("--gpus", str(gpus), "--launch-selftest")
    assert p.returncode == 0, p.stderr[-2000:]
    assert len(lines) == 1, p.stdout           # rank 0 alone prints
    assert lines[0] == {"selftest": "launch", "n_gpus": gpus, "max_rank": gpus - 1, "ranks": gpus,
                        "gpus_flag": gpus}


def test_world_size_must_match_gpus_flag():
    p, _ = run_bench("--gpus", "2", "--launch-selftest", env={"WORLD_SIZE": "1", "RANK": "0"})
    assert p.returncode != 0 and "WORLD_SIZE=1" in p.stderr


def test_reference_arm_measures_its_steps():
    import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    p, lines = run_bench("--impl", "reference", "--n", "1024", "--layout", "interleaved", "--steps", "2",
                         "--warmup", "0")
    assert p.returncode == 0, p.stderr[-2000:]
    (line,) = lines
    assert line["impl"] == "reference" and line["n_gpus"] == 0
    sample = line["config"]["sample_transforms"]
    # value and ms_per_step describe the same measured steps of `sample` transforms
    gflop = 5 * 1024 * 10 * sample / 1e9
    assert abs(gflop / (line["ms_per_step"] / 1e3) - line["value"]) / line["value"] < 0.01
    assert line["e2e"]["value"] == line["value"]
