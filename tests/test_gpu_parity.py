"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle.

Inputs are the reference's seeded_input (verify.cpp:69-78) rounded to fp32;
the oracle (oracle/fftgen_oracle.c, pinned bit-exact to the reference by
tests/test_oracle.py) transforms the same fp32-rounded values in fp64.
Tolerance (north star): fp32 relative L2 error <= 1e-5 * log2 N per
transform.  Integer / exact cases (delta, DFT_2, identity) are bit-exact.
"""
import math

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

fg = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global fg
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2308_00497_b200 as m
    fg = m
    yield


def tol(n):
    return 1e-5 * max(1.0, math.log2(n))


def seeded_batch(orc, n, batch, seed0=1):
    x = np.stack([orc.seeded_input(n, seed0 + b) for b in range(batch)])
    return x.astype(np.float32).astype(np.float64)  # fp32-rounded, widened back


def to_device(x, layout, dist=None):
    """interleaved (batch, 2n) float64 -> device tensors for the given layout."""
    batch, n2 = x.shape
    n = n2 // 2
    dist = dist or n
    if layout == "interleaved":
        buf = torch.zeros(batch, dist, 2, dtype=torch.float32, device="cuda")
        buf[:, :n, :] = torch.from_numpy(x.reshape(batch, n, 2).astype(np.float32)).cuda()
        return (buf, None)
    re = torch.zeros(batch, dist, dtype=torch.float32, device="cuda")
    im = torch.zeros(batch, dist, dtype=torch.float32, device="cuda")
    re[:, :n] = torch.from_numpy(x[:, 0::2].astype(np.float32)).cuda()
    im[:, :n] = torch.from_numpy(x[:, 1::2].astype(np.float32)).cuda()
    return (re, im)


def from_device(bufs, layout, n):
    if layout == "interleaved":
        return bufs[0][:, :n, :].reshape(bufs[0].shape[0], 2 * n).double().cpu().numpy()
    out = np.empty((bufs[0].shape[0], 2 * n))
    out[:, 0::2] = bufs[0][:, :n].double().cpu().numpy()
    out[:, 1::2] = bufs[1][:, :n].double().cpu().numpy()
    return out


def run(n, layout, direction, x, dist=None, radix=2, tuning=0, pass_radix=0):
    batch = x.shape[0]
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, radix=radix,
                                                 algorithm="stockham", tuning=tuning, pass_radix=pass_radix))
    src = to_device(x, layout, dist)
    dst = tuple(torch.full_like(t, float("nan")) if t is not None else None for t in src)
    plan.execute(src[0], dst[0], src[1], dst[1], direction=direction, dist=dist or n)
    torch.cuda.synchronize()
    return from_device(dst, layout, n)


def check(got, want, n):
    for b in range(got.shape[0]):
        err = oracle.rel_l2(got[b], want[b])
        assert err <= tol(n), (n, b, err)
    return max(oracle.rel_l2(got[b], want[b]) for b in range(got.shape[0]))


SIZES = [1 << l for l in range(0, 15)]


@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
@pytest.mark.parametrize("n", SIZES)
def test_matches_oracle_all_sizes(orc, n, layout, direction):
    batch = 3 if n >= 4096 else 5  # ragged against transforms-per-CTA
    x = seeded_batch(orc, n, batch)
    got = run(n, layout, direction, x)
    want = orc.forward(x, "stockham", 4, inverse=direction > 0)
    err = check(got, want, n)
    assert err < 2e-6, err  # fp32 quality, far inside the north-star bound


def test_reference_golden_fixtures(golden, golden_meta):
    """Outputs of the unmodified reference on fp32-rounded inputs."""
    for n, seed in golden_meta["gpu_goldens"]:
        x = golden[f"gpu_in_{n}_{seed}"].astype(np.float64)[None, :]
        want = golden[f"gpu_out_{n}_{seed}"][None, :]
        for layout in ("interleaved", "split"):
            check(run(n, layout, -1, x), want, n)


def test_known_answers_exact(orc):
    # delta -> all ones (test_exec.cpp:81-91), both directions, every size
    for n in SIZES:
        x = np.zeros((1, 2 * n))
        x[0, 0] = 1.0
        for direction in (-1, 1):
            for layout in ("interleaved", "split"):
                got = run(n, layout, direction, x)
                assert np.array_equal(got[0, 0::2], np.ones(n)), (n, layout, direction)
                assert np.array_equal(got[0, 1::2], np.zeros(n)), (n, layout, direction)
    # DFT_2(1, 2) = (3, -1) exactly (test_exec.cpp:93-99)
    got = run(2, "interleaved", -1, np.array([[1.0, 0.0, 2.0, 0.0]]))
    assert np.array_equal(got[0], [3.0, 0.0, -1.0, 0.0])
    # size-1 transform is the identity (test_cli.cpp:50-58 on seeded_input(1,0))
    x = seeded_batch(orc, 1, 4, 0)
    assert np.array_equal(run(1, "split", -1, x), x)


def test_constant_and_tone(orc):
    # constant -> N delta; single tone e^{2 pi i k0 n/N} -> N delta[k - k0]
    for n in (1024, 4096, 16384):
        k0 = 37 % n
        t = np.arange(n)
        tone = np.exp(2j * np.pi * k0 * t / n)
        x = oracle.as_interleaved(np.stack([np.ones(n, dtype=complex), tone]))
        x = x.astype(np.float32).astype(np.float64)
        got = oracle.as_complex(run(n, "split", -1, x))
        want = np.zeros((2, n), dtype=complex)
        want[0, 0] = n
        want[1, k0] = n
        assert np.abs(got - want).max() / n < 1e-5


@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_dist_larger_than_n(orc, layout):
    n = 1024
    x = seeded_batch(orc, n, 4)
    got = run(n, layout, -1, x, dist=n + 96)
    check(got, orc.forward(x, "stockham", 4), n)


def test_reference_complexbuffer_split_storage(orc):
    """Split ComplexBuffer [re n | im n] per transform: in1 = in0 + n, dist = 2n."""
    n, batch = 4096, 3
    x = seeded_batch(orc, n, batch)
    buf = torch.from_numpy(oracle.relayout_to_split(x).astype(np.float32)).cuda().contiguous()
    out = torch.empty_like(buf)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=batch))
    plan.execute(buf, out, buf[:, n:], out[:, n:], dist=2 * n)
    torch.cuda.synchronize()
    got = oracle.split_to_interleaved(out.double().cpu().numpy())
    check(got, orc.forward(x, "stockham", 4), n)


@pytest.mark.parametrize("n", [1024, 4096, 16384])
def test_roundtrip_inverse_of_forward(orc, n):
    x = seeded_batch(orc, n, 4)
    y = run(n, "interleaved", -1, x)
    z = run(n, "interleaved", 1, y.astype(np.float32).astype(np.float64)) / n
    assert oracle.rel_l2(z, x) < 1e-6


def test_bitwise_deterministic_and_layout_independent(orc):
    # test_exec.cpp:113-126 (purity); split and interleaved share the arithmetic
    n = 4096
    x = seeded_batch(orc, n, 6)
    a = run(n, "interleaved", -1, x)
    b = run(n, "interleaved", -1, x)
    c = run(n, "split", -1, x)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    # radix (reference stage list) changes introspection, not the sm_100a passes
    d = run(n, "split", -1, x, radix=8)
    assert np.array_equal(a, d)


def test_execute_host_matches_device(orc):
    n, batch = 4096, 300
    x = seeded_batch(orc, n, batch)
    want = run(n, "split", -1, x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=batch))
    re = np.ascontiguousarray(x[:, 0::2].astype(np.float32))
    im = np.ascontiguousarray(x[:, 1::2].astype(np.float32))
    ore, oim = np.empty_like(re), np.empty_like(im)
    plan.execute_host(re, ore, im, oim)
    got = np.empty_like(want)
    got[:, 0::2], got[:, 1::2] = ore, oim
    assert np.array_equal(got, want)
    # pinned host memory path
    pre = torch.from_numpy(re).pin_memory()
    pim = torch.from_numpy(im).pin_memory()
    pore, poim = torch.empty_like(pre).pin_memory(), torch.empty_like(pim).pin_memory()
    plan.execute_host(pre, pore, pim, poim)
    assert np.array_equal(pore.numpy(), ore) and np.array_equal(poim.numpy(), oim)


@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_interpret_f64_dropin(orc, layout):
    """fp64 ComplexBuffer storage in/out, like fftgen::interpret."""
    n, batch = 1024, 5
    x = seeded_batch(orc, n, batch)
    store = x if layout == "interleaved" else oracle.relayout_to_split(x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
    y = fg.interpret(plan, store)
    got = y if layout == "interleaved" else oracle.split_to_interleaved(y)
    check(got, orc.forward(x, "stockham", 4), n)
    yi = fg.interpret(plan, store, direction=fg.INVERSE)
    goti = yi if layout == "interleaved" else oracle.split_to_interleaved(yi)
    check(goti, orc.forward(x, "stockham", 4, inverse=True), n)


def test_bench_config_full_size_properties(orc):
    """N=4096, batch=65536 split (BASELINE config 2): sampled transforms vs
    the oracle plus whole-batch Parseval and linearity."""
    n, batch = 4096, 65536
    g = torch.Generator(device="cuda").manual_seed(7)
    re = torch.rand(batch, n, device="cuda", generator=g) * 2 - 1
    im = torch.rand(batch, n, device="cuda", generator=g) * 2 - 1
    ore, oim = torch.empty_like(re), torch.empty_like(im)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="split", batch=batch))
    plan.execute(re, ore, im, oim)
    torch.cuda.synchronize()
    for b in (0, 1, 12345, 40000, batch - 1):
        x = np.empty(2 * n)
        x[0::2] = re[b].double().cpu().numpy()
        x[1::2] = im[b].double().cpu().numpy()
        y = np.empty(2 * n)
        y[0::2] = ore[b].double().cpu().numpy()
        y[1::2] = oim[b].double().cpu().numpy()
        assert oracle.rel_l2(y, orc.forward(x, "stockham", 4)) < 2e-6, b
    ein = (re.double() ** 2 + im.double() ** 2).sum(dim=1)
    eout = (ore.double() ** 2 + oim.double() ** 2).sum(dim=1)
    assert torch.allclose(eout, n * ein, rtol=1e-5)


def test_execute_errors():
    plan = fg.compile_pipeline(fg.PipelineConfig(n=64, layout="split", batch=1))
    t = torch.zeros(64, device="cuda")
    with pytest.raises(fg.ExecError):
        plan.execute(t, t.clone(), t, t.clone(), direction=0)
    with pytest.raises(fg.ExecError):
        plan.execute(t, t.clone())           # split needs im pointers
    with pytest.raises(fg.DimensionError):
        plan.execute(t, t.clone(), t, t.clone(), dist=32)
    with pytest.raises(fg.PlanError):
        fg.compile_pipeline(fg.PipelineConfig(n=12))
    with pytest.raises(fg.PlanError):
        fg.compile_pipeline(fg.PipelineConfig(n=16, radix=3))
    with pytest.raises(fg.FuseError):
        fg.compile_pipeline(fg.PipelineConfig(n=256, radix=128))
    with pytest.raises(fg.DimensionError):
        fg.compile_pipeline(fg.PipelineConfig(n=16, batch=0))


def test_introspection_matches_reference_goldens(golden, golden_meta):
    for key, text in golden_meta["pipelines"].items():
        alg, n, radix = key.rsplit("_", 2)
        if int(n) > (1 << 14):
            continue
        plan = fg.compile_pipeline(fg.PipelineConfig(n=int(n), algorithm=alg, radix=int(radix)))
        assert plan.pipeline_text() == text
        for i, op in enumerate(plan.ops()):
            if f"map_{key}_{i}" in golden.files:
                m, _ = plan.op_map(i)
                assert np.array_equal(m, golden[f"map_{key}_{i}"])
    p = fg.compile_pipeline(fg.PipelineConfig(n=4096, layout="split", batch=65536))
    assert p.radices() == [2] * 12
    assert [d[0] for d in p.passes()] == [64, 64]
    assert p.launches() == 1
    assert "fft_block_tma_kernel<4096>" in p.describe()


@pytest.mark.parametrize("n", [256, 512, 1024, 2048, 4096, 8192, 16384])
def test_tma_and_direct_kernels_bitwise_equal(orc, n):
    """The persistent TMA variants (bulk-store epilogue or register stores) and
    the direct variant run the same passes: bitwise equal results."""
    x = seeded_batch(orc, n, 37)
    # 2^8 / 2^9 (radix 8) and interleaved 2^10 / 2^11 (radix 16) default to
    # three-pass direct plans; 64 keeps the two-pass TMA ones
    hint = 64 if n <= 2048 else 0
    for layout in ("interleaved", "split"):
        a = run(n, layout, -1, x, pass_radix=hint)
        b = run(n, layout, -1, x, tuning=fg.TUNE_NO_TMA, pass_radix=hint)
        c = run(n, layout, -1, x, tuning=fg.TUNE_NO_TMA_STORE, pass_radix=hint)
        assert np.array_equal(a, b) and np.array_equal(a, c), layout
        check(a, orc.forward(x, "stockham", 4), n)


@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_tma1_store_variants_bitwise_equal(orc, layout):
    """2^14 single-stage kernel with and without the bulk-store epilogue, both
    directions, over a batch of several transforms per persistent CTA."""
    n = 16384
    x = seeded_batch(orc, n, 301)
    outs = []
    for tuning in (0, fg.TUNE_NO_TMA_STORE):
        for d in (-1, 1):
            outs.append(run(n, layout, d, x, tuning=tuning))
    for i in range(2, len(outs)):
        assert np.array_equal(outs[i], outs[i % 2]), i
    check(outs[0], orc.forward(x, "stockham", 4), n)
    check(outs[1], orc.forward(x, "stockham", 4, inverse=True), n)


def test_unaligned_dist_uses_direct_path(orc):
    # dist*4 bytes not a multiple of 16 -> no cp.async.bulk; still correct
    n = 4096
    x = seeded_batch(orc, n, 5)
    check(run(n, "split", -1, x, dist=n + 3), orc.forward(x, "stockham", 4), n)
    check(run(n, "interleaved", 1, x, dist=n + 1), orc.forward(x, "stockham", 4, inverse=True), n)


def test_large_batch_persistent_grid(orc):
    """More groups than resident CTAs: every transform visited exactly once."""
    n, batch = 1024, 20000
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(batch, n, 2, device="cuda", generator=g) * 2 - 1
    y = torch.full_like(x, float("nan"))
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=batch))
    plan.execute(x, y)
    torch.cuda.synchronize()
    assert not torch.isnan(y).any()
    for b in (0, 777, batch - 1):
        xi = x[b].reshape(-1).double().cpu().numpy()
        assert oracle.rel_l2(y[b].reshape(-1).double().cpu().numpy(), orc.forward(xi, "stockham", 4)) < 2e-6


@pytest.mark.parametrize("n", [8, 16, 32, 64])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_row_kernel_small_sizes(orc, n, layout):
    """K2r (fft_rows.cu, one transform per thread, coalesced 16-byte row
    moves) for N = 8 .. 64: ragged batches (not a multiple of the CTA's
    transforms, and a single transform), padded rows (dist > N), both
    directions; a dist that breaks 16-byte alignment takes the direct kernel,
    same results within tolerance."""
    p = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=1))
    assert f"fft_rows_kernel<{n}>" in p.describe()
    assert f"fft_rows_kernel<{n}>" not in fg.compile_pipeline(
        fg.PipelineConfig(n=n, layout=layout, batch=1, tuning=fg.TUNE_NO_TMA)).describe()
    for batch in (1, 301):
        x = seeded_batch(orc, n, batch, seed0=11)
        want_f = orc.forward(x, "stockham", 4)
        want_i = orc.forward(x, "stockham", 4, inverse=True)
        for dist in (n, n + 4):
            check(run(n, layout, -1, x, dist=dist), want_f, n)
            check(run(n, layout, 1, x, dist=dist), want_i, n)
    x = seeded_batch(orc, n, 37, seed0=5)
    a = run(n, layout, -1, x, dist=n + 1)  # 4- / 8-byte row offsets: direct kernel
    b = run(n, layout, -1, x, tuning=fg.TUNE_NO_TMA)
    assert np.array_equal(a, b)
    check(a, orc.forward(x, "stockham", 4), n)
