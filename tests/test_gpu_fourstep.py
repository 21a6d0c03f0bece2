"""GPU parity of the K3 four-step path (2^15 <= N <= 2^30) vs the CPU oracle.

Same contract as tests/test_gpu_parity.py: fp32-rounded seeded inputs, the
pinned fp64 oracle (oracle/fftgen_oracle.c) on the same values, relative L2
<= 1e-5 log2 N per transform.  At sizes where a full oracle transform is too
slow, size-independent properties are used instead: single tones and
delta (analytic), sampled bins of the O(N)-per-bin dft_oracle restatement,
Parseval, and the inverse(forward) round trip.
"""
import math

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


def tol(n):
    return 1e-5 * math.log2(n)


def seeded_batch(orc, n, batch, seed0=1):
    x = np.stack([orc.seeded_input(n, seed0 + b) for b in range(batch)])
    return x.astype(np.float32).astype(np.float64)


def run(fg, n, layout, direction, x, tuning=0):
    batch = x.shape[0]
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, algorithm="stockham",
                                                 tuning=tuning))
    if layout == "interleaved":
        src = torch.from_numpy(x.astype(np.float32)).cuda()
        dst = torch.full_like(src, float("nan"))
        plan.execute(src, dst, direction=direction)
        torch.cuda.synchronize()
        return dst.double().cpu().numpy()
    re = torch.from_numpy(np.ascontiguousarray(x[:, 0::2]).astype(np.float32)).cuda()
    im = torch.from_numpy(np.ascontiguousarray(x[:, 1::2]).astype(np.float32)).cuda()
    ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
    plan.execute(re, ore, im, oim, direction=direction)
    torch.cuda.synchronize()
    out = np.empty_like(x)
    out[:, 0::2] = ore.double().cpu().numpy()
    out[:, 1::2] = oim.double().cpu().numpy()
    return out


@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
@pytest.mark.parametrize("l2", [15, 16, 17, 18, 19, 20])
def test_fourstep_matches_oracle(fg, orc, l2, layout, direction):
    n = 1 << l2
    batch = 3 if l2 <= 17 else 1
    x = seeded_batch(orc, n, batch)
    got = run(fg, n, layout, direction, x)
    want = orc.forward(x, "stockham", 4, inverse=direction > 0, threads=4)
    for b in range(batch):
        err = oracle.rel_l2(got[b], want[b])
        assert err <= tol(n) and err < 3e-6, (n, b, err)


@pytest.mark.parametrize("l2", [21, 22, 24])
def test_three_group_sizes_vs_oracle(fg, orc, l2):
    n = 1 << l2
    x = seeded_batch(orc, n, 1, seed0=5)
    got = run(fg, n, "split", -1, x, tuning=8)
    want = orc.forward(x, "stockham", 4)
    err = oracle.rel_l2(got[0], want[0])
    assert err <= tol(n) and err < 4e-6, err


@pytest.mark.parametrize("l2", [21, 22, 23, 24])
@pytest.mark.parametrize("layout,direction", [("split", -1), ("interleaved", 1)])
@pytest.mark.parametrize("tuning", [16, 16 | 1, 16 | 4])
def test_two_pass_plans_vs_oracle(fg, orc, l2, layout, direction, tuning):
    """2^21..2^24 as two groups of 2^11 / 2^12 points (plain / TMA tiles)."""
    n = 1 << l2
    batch = 2 if l2 <= 22 else 1
    x = seeded_batch(orc, n, batch, seed0=11)
    got = run(fg, n, layout, direction, x, tuning=tuning)
    want = orc.forward(x, "stockham", 4, inverse=direction > 0, threads=8)
    for b in range(batch):
        err = oracle.rel_l2(got[b], want[b])
        assert err <= tol(n) and err < 4e-6, (b, err)


def test_fourstep_plan_shape(fg):
    p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 24, layout="split", batch=1))
    assert [d[0] for d in p.passes()] == [256, 256, 256]
    assert p.launches() == 3
    assert p.scratch_bytes() == 2 * (1 << 24) * 8
    assert "transposed store" in p.describe()
    # interleaved 2^23 / 2^24 run two passes by default (NS = 2^11 / 2^12 plane kernels)
    p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 24, layout="interleaved", batch=1))
    assert [d[0] for d in p.passes()] == [4096, 4096] and "fft_group_plane_kernel<4096>" in p.describe()
    # two-pass plans: NS = 2^11 / 2^12 groups, one scratch buffer
    p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 24, layout="split", batch=1, tuning=16))
    assert [d[0] for d in p.passes()] == [4096, 4096] and p.launches() == 2
    assert p.scratch_bytes() == (1 << 24) * 8
    p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 21, layout="split", batch=1))
    assert [d[0] for d in p.passes()] == [1024, 2048] and p.launches() == 2
    p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 21, layout="split", batch=1, tuning=8))
    assert [d[0] for d in p.passes()] == [128, 128, 128]
    q = fg.compile_pipeline(fg.PipelineConfig(n=1 << 15, layout="split", batch=4))
    # 2^15 runs as one cluster per transform: one launch, no HBM intermediate;
    # the plan owns only the bounded fallback scratch for unaligned data
    assert [d[0] for d in q.passes()] == [128, 256] and q.launches() == 1
    assert q.scratch_bytes() == 4 * (1 << 15) * 8
    assert "fft_cluster_kernel<128,256,8>" in q.describe()
    q = fg.compile_pipeline(fg.PipelineConfig(n=1 << 16, layout="split", batch=4))
    assert q.launches() == 2 and q.scratch_bytes() == 4 * (1 << 16) * 8
    assert "group 0: fft_group_kernel<256>" in q.describe()
    q = fg.compile_pipeline(fg.PipelineConfig(n=1 << 18, layout="split", batch=2))
    assert [d[0] for d in q.passes()] == [1024, 256]  # measured split 10 + 8
    assert "group 0: fft_group_tma_kernel<1024>" in q.describe()


def test_fourstep_host_and_interpret_paths(fg, orc):
    n, batch = 1 << 15, 5
    x = seeded_batch(orc, n, batch)
    want = orc.forward(x, "stockham", 4, threads=4)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=batch))
    re = np.ascontiguousarray(x[:, 0::2].astype(np.float32))
    im = np.ascontiguousarray(x[:, 1::2].astype(np.float32))
    ore, oim = np.empty_like(re), np.empty_like(im)
    plan.execute_host(re, ore, im, oim)
    got = np.empty_like(x)
    got[:, 0::2], got[:, 1::2] = ore, oim
    for b in range(batch):
        assert oracle.rel_l2(got[b], want[b]) < 3e-6
    y = fg.interpret(plan, oracle.relayout_to_split(x))
    assert oracle.rel_l2(oracle.split_to_interleaved(y), want) < 3e-6


@pytest.mark.parametrize("l2", [26, 30])
def test_huge_single_transform_tones(fg, l2):
    """N = 2^26 .. 2^30: x = e^{2 pi i k1 n/N} + 0.5 e^{-2 pi i k2 n/N}
    -> X = N delta[k - k1] + N/2 delta[k + k2] (forward), exact analytic answer."""
    n = 1 << l2
    k1, k2 = 12345, 987654 % n
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    ph1 = ((idx * k1) % n).double() * (2 * math.pi / n)
    ph2 = ((idx * k2) % n).double() * (-2 * math.pi / n)
    re = (torch.cos(ph1) + 0.5 * torch.cos(ph2)).float()
    im = (torch.sin(ph1) + 0.5 * torch.sin(ph2)).float()
    del idx, ph1, ph2
    ore, oim = torch.empty_like(re), torch.empty_like(im)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=1))
    plan.execute(re, ore, im, oim)
    torch.cuda.synchronize()
    ore[k1] -= n
    ore[(n - k2) % n] -= n / 2
    err = torch.sqrt((ore.double() ** 2 + oim.double() ** 2).max()).item() / n
    assert err < 1e-5, err
    plan.close()


def test_2p26_random_sampled_bins_and_roundtrip(fg, orc):
    n = 1 << 26
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.rand(n, 2, device="cuda", generator=g) * 2 - 1).contiguous()
    y = torch.empty_like(x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=1))
    plan.execute(x, y)
    z = torch.empty_like(x)
    plan.execute(y, z, direction=fg.INVERSE)
    torch.cuda.synchronize()
    assert torch.linalg.norm((z / n - x).double()) / torch.linalg.norm(x.double()) < 1e-6
    # Parseval
    ex = (x.double() ** 2).sum()
    ey = (y.double() ** 2).sum()
    assert abs(ey / (n * ex) - 1) < 1e-6
    # sampled bins of the O(N)-per-bin oracle restatement
    xh = x.reshape(-1).double().cpu().numpy()
    bins = [0, 1, 777, n // 2, n - 1]
    want = orc.dft_bins(xh, bins)
    got = np.concatenate([y[b].double().cpu().numpy() for b in bins])
    scale = math.sqrt(n)  # typical |X| for unit-variance random input
    assert np.abs(got - want).max() / scale < 1e-4


@pytest.mark.parametrize("l2,batch,csize", [(15, 301, 4), (15, 301, 8), (16, 150, 8), (16, 150, 16)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
def test_cluster_kernel_bitwise_two_launch_path(fg, orc, l2, batch, csize, layout, direction):
    """K5 (persistent clusters, one transform per cluster, TMA tensor tiles in,
    the intermediate exchanged through distributed shared memory) performs
    exactly the arithmetic of the two-launch K3 path, so the results are
    bitwise equal for every compiled cluster size; both match the oracle."""
    n = 1 << l2
    g = torch.Generator(device="cuda").manual_seed(100 + l2)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1

    def run_once(cluster_size):
        plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, cluster_size=cluster_size))
        if layout == "interleaved":
            y = torch.full_like(x, float("nan"))
            plan.execute(x, y, direction=direction)
        else:
            re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
            ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
            plan.execute(re, ore, im, oim, direction=direction)
            y = torch.stack([ore, oim], dim=-1)
        torch.cuda.synchronize()
        return y, plan.describe()

    cl, d1 = run_once(csize)
    assert f"fft_cluster_kernel<{1 << (l2 // 2)},{1 << (l2 - l2 // 2)},{csize}>" in d1
    two, d2 = run_once(-1)
    assert "fft_cluster_kernel" not in d2
    assert torch.equal(cl, two)
    for b in (0, batch // 2, batch - 1):
        xi = x[b].reshape(-1).double().cpu().numpy()
        got = cl[b].reshape(-1).double().cpu().numpy()
        want = orc.forward(xi, "stockham", 4, inverse=direction > 0)
        assert oracle.rel_l2(got, want) < 3e-6, b


def test_cluster_kernel_unaligned_rows_fall_back(fg, orc):
    """TMA tensor tiles need 16-byte aligned rows: an odd element offset runs
    the two-launch path (in chunks through the plan's bounded fallback
    scratch), with the same result."""
    n, batch = 1 << 15, 9
    g = torch.Generator(device="cuda").manual_seed(5)
    buf = torch.rand(batch * n * 2 + 2, device="cuda", generator=g) * 2 - 1
    x = buf[2:].view(batch, n, 2)                    # 8-byte offset: not 16-byte aligned
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="interleaved", batch=batch))
    assert "fft_cluster_kernel" in plan.describe()
    y = torch.full((batch, n, 2), float("nan"), device="cuda")
    plan.execute(x, y)
    aligned = x.clone()
    y2 = torch.full_like(y, float("nan"))
    plan.execute(aligned, y2)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    want = orc.forward(x[3].reshape(-1).double().cpu().numpy(), "stockham", 4)
    assert oracle.rel_l2(y[3].reshape(-1).double().cpu().numpy(), want) < 3e-6


@pytest.mark.parametrize("l2,batch", [(15, 40), (16, 20), (18, 6), (20, 3), (21, 2), (22, 1), (28, 1)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_group_tma_kernels_bitwise_plain(fg, orc, l2, batch, layout):
    """The persistent TMA group kernels (tensor-tile prefetch) are bitwise the
    plain group kernels for every shape (first / middle columns, rows)."""
    if l2 == 28 and layout == "interleaved":
        pytest.skip("one layout suffices at 2^28")
    n = 1 << l2
    g = torch.Generator(device="cuda").manual_seed(l2)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1

    def run_once(tma):
        tuning = fg.TUNE_GROUP_TMA_ALL if tma == "1" else fg.TUNE_NO_TMA
        plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, cluster_size=-1,
                                                     tuning=tuning))
        if layout == "interleaved":
            y = torch.full_like(x, float("nan"))
            plan.execute(x, y)
        else:
            re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
            ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
            plan.execute(re, ore, im, oim)
            y = torch.stack([ore, oim], dim=-1)
        torch.cuda.synchronize()
        d = plan.describe()
        plan.close()
        return y, d

    a, da = run_once("1")
    assert "fft_group_tma_kernel" in da or "fft_group_plane_kernel" in da
    b, db = run_once("0")
    assert "fft_group_tma_kernel" not in db and "fft_group_plane_kernel" not in db
    assert torch.equal(a, b)
    if l2 <= 20:
        xi = x[0].reshape(-1).double().cpu().numpy()
        assert oracle.rel_l2(a[0].reshape(-1).double().cpu().numpy(), orc.forward(xi, "stockham", 4)) < 3e-6


@pytest.mark.parametrize("l2", [21, 22])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_three_group_inverse_vs_oracle(fg, orc, l2, layout):
    """Inverse (conjugate-root) instances of the first / middle / last group
    kernels of a 3-group plan against the oracle."""
    n = 1 << l2
    x = seeded_batch(orc, n, 1, seed0=9)
    got = run(fg, n, layout, 1, x)
    want = orc.forward(x, "stockham", 4, inverse=True)
    assert oracle.rel_l2(got[0], want[0]) <= tol(n)


@pytest.mark.parametrize("l2", [28, 30])
def test_huge_roundtrip_inverse(fg, l2):
    """inverse(forward(x)) / N == x at 2^28 (3 groups) and 2^30 (4 groups):
    the inverse instances of every group shape on the largest plans."""
    n = 1 << l2
    g = torch.Generator(device="cuda").manual_seed(l2)
    x = torch.rand(n, 2, device="cuda", generator=g) * 2 - 1
    y = torch.empty_like(x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=1))
    plan.execute(x, y)
    plan.execute(y, y, direction=fg.INVERSE)  # in place
    torch.cuda.synchronize()
    err = (torch.linalg.norm((y / n - x).double()) / torch.linalg.norm(x.double())).item()
    assert err < 1e-6, err
    plan.close()
