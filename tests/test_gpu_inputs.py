"""The device-side seeded_input (fftgen_seeded_input, verify.cpp:55-78) and the
headline configuration C2 run on it: N=4096, batch 65536, split -- every one
of the 65536 transforms checked against the pinned oracle."""
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    assert torch.cuda.is_available()
    import paper_2308_00497_b200 as m
    return m


@pytest.mark.parametrize("n,batch,seed0", [(1, 3, 1), (1024, 5, 1), (4096, 7, 1000), (1 << 16, 2, 2 ** 40)])
def test_seeded_input_bitwise_the_host_generator(fg, orc, n, batch, seed0):
    want = np.stack([orc.seeded_input(n, seed0 + b) for b in range(batch)]).astype(np.float32)
    x = fg.seeded_input(n, batch, "interleaved", seed0=seed0)
    assert np.array_equal(x.cpu().numpy().reshape(batch, 2 * n), want)
    re, im = fg.seeded_input(n, batch, "split", seed0=seed0, dist=n + 3)
    assert np.array_equal(re[:, :n].cpu().numpy(), want[:, 0::2])
    assert np.array_equal(im[:, :n].cpu().numpy(), want[:, 1::2])


def test_seeded_input_validation(fg):
    with pytest.raises(fg.DimensionError):
        fg.seeded_input(16, 2, dist=8)


def test_c2_full_batch_on_reference_inputs_vs_oracle(fg, orc):
    """BASELINE configs[1] exactly as bench.py runs it: inputs from the device
    generator (seeds 1..65536), one execute, all 65536 outputs vs the oracle."""
    n, batch = 4096, 65536
    re, im = fg.seeded_input(n, batch, "split", seed0=1)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=batch, algorithm="stockham"))
    ore, oim = torch.empty_like(re), torch.empty_like(im)
    plan.execute(re, ore, im, oim)
    torch.cuda.synchronize()
    del re, im
    threads = os.cpu_count() or 4
    chunk = 4096
    worst = 0.0
    for b0 in range(0, batch, chunk):
        x = np.stack([orc.seeded_input(n, 1 + b) for b in range(b0, b0 + chunk)])
        x = x.astype(np.float32).astype(np.float64)
        want = orc.forward(x, "stockham", 4, threads=threads)
        got = np.empty_like(want)
        got[:, 0::2] = ore[b0:b0 + chunk].double().cpu().numpy()
        got[:, 1::2] = oim[b0:b0 + chunk].double().cpu().numpy()
        err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
        worst = max(worst, float(err.max()))
    assert worst <= 1e-5 * 12 and worst < 2e-6, worst
