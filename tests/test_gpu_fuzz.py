"""Randomised GPU parity across every execution strategy.

A fixed-seed list of (N, batch, dist padding, layout, direction) cases drawn
over N = 2^0 .. 2^20, so that batch counts that are not multiples of a CTA's
transforms, padded and unaligned distances (which switch TMA paths to their
direct / two-launch fallbacks) and every plan shape (identity, K2 direct and
TMA, K5 cluster, K3 two- and three-group) meet the oracle.  Tolerance as in
test_gpu_parity.py: relative L2 <= 1e-5 log2 N (and < 3e-6) per transform.
"""
import math
import random

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def cases():
    rnd = random.Random(20231017)
    out = []
    for l2 in range(0, 21):
        for _ in range(2):
            n = 1 << l2
            max_batch = max(1, min(37, (1 << 22) // max(n, 1)))
            batch = rnd.randint(1, max_batch)
            pad = rnd.choice([0, 0, 1, 2, 3, 8, 64])
            out.append((n, batch, n + pad, rnd.choice(["interleaved", "split"]), rnd.choice([-1, 1])))
    return out


@pytest.fixture(scope="module")
def fg():
    import paper_2308_00497_b200 as m
    return m


@pytest.mark.parametrize("n,batch,dist,layout,direction", cases())
def test_random_geometry_matches_oracle(fg, orc, n, batch, dist, layout, direction):
    g = torch.Generator(device="cuda").manual_seed(n * 1000 + batch)
    x = (torch.rand(batch, dist, 2, device="cuda", generator=g) * 2 - 1).contiguous()
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
    if layout == "interleaved":
        y = torch.full_like(x, float("nan"))
        plan.execute(x, y, direction=direction, dist=dist)
    else:
        re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
        ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
        plan.execute(re, ore, im, oim, direction=direction, dist=dist)
        y = torch.stack([ore, oim], dim=-1)
    torch.cuda.synchronize()
    tol = min(3e-6, 1e-5 * max(1.0, math.log2(n)))
    for b in sorted({0, batch // 2, batch - 1}):
        xi = x[b, :n].reshape(-1).double().cpu().numpy()
        got = y[b, :n].reshape(-1).double().cpu().numpy()
        want = orc.forward(xi, "stockham", 4, inverse=direction > 0)
        if n == 1:
            assert np.array_equal(got, xi)
        else:
            assert oracle.rel_l2(got, want) <= tol, (n, batch, dist, layout, direction, b)
    # the padding between transforms is never written
    if dist > n:
        assert torch.isnan(y[:, n:]).all()
    plan.close()
