"""GPU edge cases across the execution strategies: in-place execution,
CUDA-graph capture and replay, ragged batches and padded dist on the
four-step path, unaligned pointers, and plan reuse across batch sizes."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    import paper_2308_00497_b200 as m
    return m


def rand(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(*shape, device="cuda", generator=g) * 2 - 1


def check_rows(orc, x, y, n, inverse=False, rows=(0, -1)):
    """x, y: (batch, n, 2) float32 device tensors."""
    for b in rows:
        xi = x[b].reshape(-1).double().cpu().numpy()
        got = y[b].reshape(-1).double().cpu().numpy()
        assert oracle.rel_l2(got, orc.forward(xi, "stockham", 4, inverse=inverse)) < 3e-6, b


@pytest.mark.parametrize("n", [1024, 4096, 16384, 1 << 15, 1 << 16, 1 << 18, 1 << 21])
def test_in_place_execution(fg, orc, n):
    batch = 4 if n <= 1 << 16 else 1
    x = rand((batch, n, 2), 1)
    ref = x.clone()
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch))
    plan.execute(x, x)  # out == in
    torch.cuda.synchronize()
    check_rows(orc, ref, x, n)
    re, im = ref[..., 0].contiguous(), ref[..., 1].contiguous()
    ps = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch, layout="split"))
    ps.execute(re, re, im, im, direction=fg.INVERSE)
    torch.cuda.synchronize()
    check_rows(orc, ref, torch.stack([re, im], -1), n, inverse=True)


@pytest.mark.parametrize("n", [1024, 4096, 8192, 16384, 1 << 15])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_in_place_persistent_kernels_many_transforms(fg, orc, n, layout):
    """In-place with several transforms per persistent CTA / cluster: the
    prefetch of transform b + grid never reads what the bulk stores of
    transform b write."""
    batch = 450
    x = rand((batch, n, 2), 7)
    ref = x.clone()
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch, layout=layout))
    if layout == "interleaved":
        plan.execute(x, x)
        y = x
    else:
        re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
        plan.execute(re, re, im, im)
        y = torch.stack([re, im], -1)
    torch.cuda.synchronize()
    check_rows(orc, ref, y, n, rows=(0, 147, 148, 296, batch - 1))


@pytest.mark.parametrize("n", [4096, 16384, 1 << 15, 1 << 16, 1 << 18])
def test_cuda_graph_capture_and_replay(fg, orc, n):
    batch = 64
    x = rand((batch, n, 2), 2)
    y = torch.empty_like(x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.execute(x, y, stream=s)  # warm-up outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.execute(x, y, stream=s)
    y.zero_()
    x.copy_(rand((batch, n, 2), 3))
    g.replay()
    torch.cuda.synchronize()
    check_rows(orc, x, y, n, rows=(0, 17, batch - 1))


@pytest.mark.parametrize("n", [1 << 15, 1 << 16])
def test_cluster_in_place_and_graph(fg, orc, n):
    """K5: in place is safe (each transform's tiles are read before any of its
    outputs is written) and the persistent launch replays from a CUDA graph.
    Unaligned data takes the two-launch path through the plan's bounded
    fallback scratch (allocated with the plan): it captures and replays too."""
    batch = 200
    x = rand((batch, n, 2), 6)
    ref = x.clone()
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch, cluster_size=8 if n == 1 << 15 else 16))
    assert "fft_cluster_kernel" in plan.describe()
    plan.execute(x, x)
    torch.cuda.synchronize()
    check_rows(orc, ref, x, n, rows=(0, 99, batch - 1))
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.execute(ref, y, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.execute(ref, y, stream=s)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    check_rows(orc, ref, y, n, rows=(1, batch - 2))
    # the fallback scratch: <= 64 MiB, whole transforms, owned by the plan
    assert 0 < plan.scratch_bytes() <= 64 << 20 and plan.scratch_bytes() % (n * 8) == 0
    buf = torch.zeros(batch * n * 2 + 2, device="cuda")
    unaligned = buf[2:].view(batch, n, 2)
    unaligned.copy_(ref)
    y2 = torch.full_like(y, float("nan"))
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        plan.execute(unaligned, y2, stream=s)
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, y2)  # chunked two-launch path == cluster kernel, bitwise


@pytest.mark.parametrize("n", [1 << 15, 1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 22, 1 << 23])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_fourstep_ragged_batch_and_padded_dist(fg, orc, n, layout):
    """Padded rows through every K3 epilogue: register stores, the TMA tensor
    stores of the NS = 512 / 1024 rows and split NS = 1024 columns, the
    plane kernels' staged halves (2^22, 2^23)."""
    batch, dist = 3, n + 64
    x = rand((batch, dist, 2), 4)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch, layout=layout))
    if layout == "interleaved":
        y = torch.full_like(x, float("nan"))
        plan.execute(x, y, dist=dist)
    else:
        re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
        ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
        plan.execute(re, ore, im, oim, dist=dist)
        y = torch.stack([ore, oim], -1)
    torch.cuda.synchronize()
    assert torch.isnan(y[:, n:]).all()  # padding untouched
    check_rows(orc, x[:, :n], y[:, :n], n, rows=(0, 1, 2))


def test_unaligned_pointers_fall_back_to_direct_kernel(fg, orc):
    n, batch = 4096, 5
    buf = rand((batch * n * 2 + 4,), 5)
    x = buf[2:2 + batch * n * 2].view(batch, n, 2)  # 8-byte aligned, not 16: no cp.async.bulk
    out = torch.empty(batch * n * 2 + 4, device="cuda")
    y = out[2:2 + batch * n * 2].view(batch, n, 2)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch))
    plan.execute(x, y)
    torch.cuda.synchronize()
    check_rows(orc, x, y, n, rows=(0, 4))
    # a float2 stream that is not even 8-byte aligned is rejected, not faulted
    with pytest.raises(fg.ExecError):
        plan.execute(buf[1:1 + batch * n * 2], y)


def test_fourstep_store_epilogues_per_group(fg):
    """The plan states which K3 groups leave by TMA tensor stores (the
    measured rule of fft_group_tma.cuh: NS = 512 / 2^19's NS = 1024 rows,
    split-input NS = 1024 columns, plane-kernel columns, NS = 4096 rows and
    NS = 2048 rows of split output)."""
    def stores(n, layout):
        d = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=1)).describe()
        return [("results by TMA tensor stores" in ln) for ln in d.splitlines() if ln.startswith("  group ")]
    # 2^18 as 10 + 8, 2^19 as 10 + 9 (split) / 11 + 8 (interleaved), 2^20 interleaved as 12 + 8
    assert stores(1 << 18, "split") == [True, False] and stores(1 << 18, "interleaved") == [False, False]
    assert stores(1 << 19, "split") == [True, True] and stores(1 << 19, "interleaved") == [True, False]
    assert stores(1 << 20, "split") == [True, False] and stores(1 << 20, "interleaved") == [True, False]
    assert stores(1 << 17, "split") == [False, False]
    assert stores(1 << 22, "split") == [True, True] and stores(1 << 22, "interleaved") == [True, False]
    assert stores(1 << 24, "interleaved") == [True, True] and stores(1 << 16, "split") == [False, False]


@pytest.mark.parametrize("n", [1 << 18, 1 << 20, 1 << 23])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_fourstep_unaligned_output_falls_back(fg, orc, n, layout):
    """An output that is 8- but not 16-byte aligned cannot be a TMA tensor
    store target: those groups take the register-store kernels, same results."""
    batch = 2
    x = rand((batch, n, 2), 9)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch, layout=layout))
    if layout == "interleaved":
        out = torch.full((batch * n * 2 + 4,), float("nan"), device="cuda")
        y = out[2:2 + batch * n * 2].view(batch, n, 2)
        plan.execute(x, y)
        yy = torch.empty_like(x)
        plan.execute(x, yy)
    else:
        re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
        out = torch.full((2, batch * n + 4), float("nan"), device="cuda")
        ore, oim = out[0, 1:1 + batch * n].view(batch, n), out[1, 1:1 + batch * n].view(batch, n)
        plan.execute(re, ore, im, oim)
        y = torch.stack([ore, oim], -1)
        a, b = torch.empty_like(re), torch.empty_like(im)
        plan.execute(re, a, im, b)
        yy = torch.stack([a, b], -1)
    torch.cuda.synchronize()
    assert torch.equal(y, yy)  # the store epilogue does not change the arithmetic
    check_rows(orc, x, y, n, rows=(0, 1))


def test_smaller_batch_than_planned_via_host_path(fg, orc):
    """execute_host chunks a plan's batch; the last chunk is ragged."""
    n, batch = 1 << 16, 257  # 128 MiB chunks of 128 transforms, ramped head and tail
    x = np.random.default_rng(0).uniform(-1, 1, (batch, n * 2)).astype(np.float32)
    y = np.empty_like(x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch))
    plan.execute_host(x, y)
    for b in (0, 63, 64, 256):
        assert oracle.rel_l2(y[b], orc.forward(x[b].astype(np.float64), "stockham", 4)) < 3e-6


def test_many_plans_and_destroy(fg):
    plans = [fg.compile_pipeline(fg.PipelineConfig(n=1 << l, batch=2)) for l in range(1, 21)]
    for p in plans:
        assert p.launches() >= 1
        p.close()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        p = fg.compile_pipeline(fg.PipelineConfig(n=1 << 20, batch=16))
        p.close()
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)  # no leak of scratch/tables


def test_partial_overlap_rejected_exact_in_place_accepted(fg, orc):
    """validate_exec: an output plane sharing bytes with an input plane is an
    ExecError unless it is exactly in place; the reference's [re n | im n]
    storage (in1 = in0 + n, dist = 2n) in place is two disjoint strided sets."""
    n, batch = 1024, 3
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch))
    buf = rand(((batch + 1) * n + 64, 2), 4)
    with pytest.raises(fg.ExecError, match="overlaps"):
        plan.execute(buf[:batch * n], buf[32:32 + batch * n])       # shifted by 32 elements
    with pytest.raises(fg.ExecError, match="overlaps"):
        plan.execute(buf[:batch * n], buf[n:n + batch * n])         # shifted by one transform
    ref = buf[:batch * n].clone()
    plan.execute(buf[:batch * n], buf[:batch * n])                  # exactly in place
    torch.cuda.synchronize()
    check_rows(orc, ref.view(batch, n, 2), buf[:batch * n].view(batch, n, 2), n, rows=(0, 2))
    sp = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch, layout="split"))
    blk = rand((batch, 2 * n), 5)
    want = blk.clone()
    sp.execute(blk, blk, blk[:, n:], blk[:, n:], dist=2 * n)       # [re n | im n] in place
    out = torch.empty_like(want)
    sp.execute(want, out, want[:, n:], out[:, n:], dist=2 * n)
    torch.cuda.synchronize()
    assert torch.equal(blk, out)
    with pytest.raises(fg.ExecError, match="overlap"):
        sp.execute(want, out, want[:, n:], out[:, 1:], dist=2 * n)  # im plane over the re plane
