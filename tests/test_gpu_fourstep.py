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


def run(fg, n, layout, direction, x):
    batch = x.shape[0]
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, algorithm="stockham"))
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
    got = run(fg, n, "split", -1, x)
    want = orc.forward(x, "stockham", 4)
    err = oracle.rel_l2(got[0], want[0])
    assert err <= tol(n) and err < 4e-6, err


def test_fourstep_plan_shape(fg):
    p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 24, layout="split", batch=1))
    assert [d[0] for d in p.passes()] == [256, 256, 256]
    assert p.launches() == 3
    assert p.scratch_bytes() == 2 * (1 << 24) * 8
    assert "transposed store" in p.describe()
    q = fg.compile_pipeline(fg.PipelineConfig(n=1 << 15, layout="split", batch=4))
    # 2^15 runs as one cluster per transform: one launch, no HBM scratch
    assert [d[0] for d in q.passes()] == [128, 256] and q.scratch_bytes() == 0 and q.launches() == 1
    assert "fft_cluster_kernel<128,256,8>" in q.describe()
    q = fg.compile_pipeline(fg.PipelineConfig(n=1 << 16, layout="split", batch=4))
    assert q.launches() == 2 and q.scratch_bytes() == 4 * (1 << 16) * 8
    assert "group 0: fft_group_kernel<256>" in q.describe()
    q = fg.compile_pipeline(fg.PipelineConfig(n=1 << 18, layout="split", batch=2))
    assert "group 0: fft_group_tma_kernel<512>" in q.describe()


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


@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_l2_chunked_two_group_path(fg, orc, layout, monkeypatch):
    """Batched 2-group plans run in L2-sized chunks on two internal streams;
    the result is bitwise the unchunked one and matches the oracle."""
    n, batch = 1 << 15, 700   # chunk = 32 MiB / 256 KiB = 128 transforms -> 6 chunks
    g = torch.Generator(device="cuda").manual_seed(21)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1

    def run_once():
        plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
        if layout == "interleaved":
            y = torch.full_like(x, float("nan"))
            plan.execute(x, y)
        else:
            re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
            ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
            plan.execute(re, ore, im, oim)
            y = torch.stack([ore, oim], dim=-1)
        torch.cuda.synchronize()
        return y

    monkeypatch.setenv("FFTGEN_DISABLE_CLUSTER", "1")
    monkeypatch.setenv("FFTGEN_PHASED", "0")
    monkeypatch.setenv("FFTGEN_L2_CHUNK_BYTES", str(32 << 20))
    chunked = run_once()
    monkeypatch.setenv("FFTGEN_L2_CHUNK_BYTES", "0")
    plain = run_once()
    monkeypatch.delenv("FFTGEN_L2_CHUNK_BYTES")
    assert torch.equal(chunked, plain)
    for b in (0, 127, 128, 555, batch - 1):
        xi = x[b].reshape(-1).double().cpu().numpy()
        got = chunked[b].reshape(-1).double().cpu().numpy()
        assert oracle.rel_l2(got, orc.forward(xi, "stockham", 4)) < 3e-6, b


@pytest.mark.parametrize("l2,batch,csize", [(14, 301, 2), (14, 301, 4), (15, 301, 4), (15, 301, 8),
                                            (16, 150, 8), (16, 150, 16)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
def test_cluster_kernel_bitwise_two_launch_path(fg, orc, l2, batch, csize, layout, direction, monkeypatch):
    """K5 (persistent clusters, one transform per cluster, TMA tensor tiles in,
    the intermediate exchanged through distributed shared memory) performs
    exactly the arithmetic of the two-launch K3 path, so the results are
    bitwise equal for every compiled cluster size; both match the oracle."""
    n = 1 << l2
    g = torch.Generator(device="cuda").manual_seed(100 + l2)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1
    if l2 == 14:
        monkeypatch.setenv("FFTGEN_CLUSTER14", "1")  # plan 2^14 as 2^7 x 2^7 groups

    def run_once():
        plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
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

    monkeypatch.setenv("FFTGEN_CLUSTER_SIZE", str(csize))
    cl, d1 = run_once()
    assert f"fft_cluster_kernel<{1 << (l2 // 2)},{1 << (l2 - l2 // 2)},{csize}>" in d1
    monkeypatch.delenv("FFTGEN_CLUSTER_SIZE")
    monkeypatch.setenv("FFTGEN_DISABLE_CLUSTER", "1")
    two, d2 = run_once()
    assert "fft_cluster_kernel" not in d2
    assert torch.equal(cl, two)
    for b in (0, batch // 2, batch - 1):
        xi = x[b].reshape(-1).double().cpu().numpy()
        got = cl[b].reshape(-1).double().cpu().numpy()
        want = orc.forward(xi, "stockham", 4, inverse=direction > 0)
        assert oracle.rel_l2(got, want) < 3e-6, b


def test_cluster_kernel_unaligned_rows_fall_back(fg, orc):
    """TMA tensor tiles need 16-byte aligned rows: an odd element offset runs
    the two-launch path on lazily allocated scratch, with the same result."""
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


@pytest.mark.parametrize("l2,batch", [(15, 40), (16, 20), (18, 6), (20, 3), (22, 1), (28, 1)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_group_tma_kernels_bitwise_plain(fg, orc, l2, batch, layout, monkeypatch):
    """The persistent TMA group kernels (tensor-tile prefetch) are bitwise the
    plain group kernels for every shape (first / middle columns, rows)."""
    if l2 == 28 and layout == "interleaved":
        pytest.skip("one layout suffices at 2^28")
    n = 1 << l2
    g = torch.Generator(device="cuda").manual_seed(l2)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1
    monkeypatch.setenv("FFTGEN_DISABLE_CLUSTER", "1")
    monkeypatch.setenv("FFTGEN_PHASED", "0")

    def run_once(tma):
        monkeypatch.setenv("FFTGEN_GROUP_TMA", tma)
        plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
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
    assert "fft_group_tma_kernel" in da
    b, db = run_once("0")
    assert "fft_group_tma_kernel" not in db
    assert torch.equal(a, b)
    if l2 <= 20:
        xi = x[0].reshape(-1).double().cpu().numpy()
        assert oracle.rel_l2(a[0].reshape(-1).double().cpu().numpy(), orc.forward(xi, "stockham", 4)) < 3e-6


@pytest.mark.parametrize("l2,batch,slot_mb", [(15, 301, 24), (15, 37, 1), (16, 150, 24), (16, 9, 1),
                                              (17, 77, 3), (18, 20, 24), (19, 7, 8), (20, 5, 8), (20, 2, 24)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
@pytest.mark.parametrize("variant,lag", [("1", "1"), ("2", "1"), ("2", "3")])
def test_phased_kernel_bitwise_two_launch_path(fg, orc, l2, batch, slot_mb, layout, direction, variant, lag,
                                               monkeypatch):
    """K6 (both groups in one cooperative launch, chunks alternating between two
    L2-resident slots, grid barrier per chunk, intermediate discarded after use)
    (opt-in) is bitwise the two-launch K3 path, for ragged last chunks, one-transform
    chunks and batches smaller than a chunk; both match the oracle."""
    n = 1 << l2
    g = torch.Generator(device="cuda").manual_seed(200 + l2)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1
    monkeypatch.setenv("FFTGEN_DISABLE_CLUSTER", "1")
    monkeypatch.setenv("FFTGEN_PHASED", variant)
    monkeypatch.setenv("FFTGEN_PHASE_LAG", lag)
    monkeypatch.setenv("FFTGEN_PHASE_SLOT_MB", str(slot_mb))

    def run_once():
        plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
        if layout == "interleaved":
            y = torch.full_like(x, float("nan"))
            plan.execute(x, y, direction=direction)
        else:
            re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
            ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
            plan.execute(re, ore, im, oim, direction=direction)
            y = torch.stack([ore, oim], dim=-1)
        torch.cuda.synchronize()
        d = plan.describe()
        plan.close()
        return y, d

    ph, d1 = run_once()
    assert ("fft_phased_kernel" if variant == "1" else "fft_stream_kernel") in d1
    monkeypatch.setenv("FFTGEN_PHASED", "0")
    two, d2 = run_once()
    assert "fft_phased_kernel" not in d2 and "fft_stream_kernel" not in d2
    assert torch.equal(ph, two)
    for b in (0, batch - 1):
        xi = x[b].reshape(-1).double().cpu().numpy()
        want = orc.forward(xi, "stockham", 4, inverse=direction > 0)
        assert oracle.rel_l2(ph[b].reshape(-1).double().cpu().numpy(), want) < 3e-6, b


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


@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
@pytest.mark.parametrize("l2", [15, 16])
def test_split_cluster_kernel_matches_oracle(fg, orc, l2, layout, direction, monkeypatch):
    """K7 (fft_split.cuh): radix-C DIF step across a C-CTA cluster, one
    2^14-point transform per CTA.  A batch above the co-resident cluster count
    exercises the persistent loop (raw slice refills, z mbarrier phases)."""
    monkeypatch.setenv("FFTGEN_SPLIT", "1")
    n = 1 << l2
    batch = 5
    x = seeded_batch(orc, n, batch, seed0=11)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
    assert "fft_split_kernel" in plan.describe() and plan.launches() == 1
    plan.close()
    got = run(fg, n, layout, direction, x)
    want = orc.forward(x, "stockham", 4, inverse=direction > 0, threads=4)
    for b in range(batch):
        err = oracle.rel_l2(got[b], want[b])
        assert err <= tol(n) and err < 3e-6, (n, b, err)


@pytest.mark.parametrize("l2", [15, 16])
def test_split_cluster_kernel_long_batch(fg, orc, l2, monkeypatch):
    """Many transforms per cluster: forward then inverse round trip on a batch
    several times the co-resident cluster count, plus oracle spot checks."""
    monkeypatch.setenv("FFTGEN_SPLIT", "1")
    n = 1 << l2
    batch = 300
    g = torch.Generator(device="cuda").manual_seed(l2)
    x = (torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1).contiguous()
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="interleaved", batch=batch))
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    plan.execute(x, y, direction=-1)
    plan.execute(y, z, direction=1)
    torch.cuda.synchronize()
    err = ((z / n - x).norm() / x.norm()).item()
    assert err < 1e-6, err
    for b in (0, 137, batch - 1):
        xi = x[b].reshape(-1).double().cpu().numpy()
        want = orc.forward(xi[None], "stockham", 4, threads=4)[0]
        assert oracle.rel_l2(y[b].reshape(-1).double().cpu().numpy(), want) <= tol(n), b
    plan.close()


def test_split_cluster_unaligned_falls_back(fg, orc, monkeypatch):
    monkeypatch.setenv("FFTGEN_SPLIT", "1")
    n = 1 << 15
    x = seeded_batch(orc, n, 2, seed0=3)
    dist = n + 1
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=2))
    xs = np.zeros((2, dist, 2))
    xs[:, :n, 0], xs[:, :n, 1] = x[:, 0::2], x[:, 1::2]
    re = torch.from_numpy(xs[..., 0].astype(np.float32)).cuda()
    im = torch.from_numpy(xs[..., 1].astype(np.float32)).cuda()
    ore, oim = torch.zeros_like(re), torch.zeros_like(im)
    plan.execute(re, ore, im, oim, direction=-1, dist=dist)
    torch.cuda.synchronize()
    got = np.empty((2, 2 * n))
    got[:, 0::2], got[:, 1::2] = ore[:, :n].double().cpu().numpy(), oim[:, :n].double().cpu().numpy()
    want = orc.forward(x, "stockham", 4)
    for b in range(2):
        assert oracle.rel_l2(got[b], want[b]) <= tol(n)
    plan.close()
