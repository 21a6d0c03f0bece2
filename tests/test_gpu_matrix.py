"""The matrix every kernel path executes, entry by entry.

A batch of impulses delta[n - b] through a plan yields the rows of the matrix
the kernels apply; it must be the DFT matrix F[b][k] = w_N^{b k}
(forward w = exp(-2 pi i / N), unit_root, matrix.cpp:14-35; inverse its
conjugate).  Every output element of an impulse is one product of twiddles
routed through the pass structure, so a wrong gather / scatter address or
twiddle index anywhere in the executed schedule -- the folded FusedPKIV /
Permute / TwiddleMul of SURVEY 8(a) a9-a11 -- shows up as an O(1) error in
some entry.  For N <= 2^14 the whole N x N matrix is checked (every
executed address); beyond, full rows for a set of impulse positions.
Tolerance: |error| <= 2e-6 per entry (entries have modulus 1).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    assert torch.cuda.is_available()
    import paper_2308_00497_b200 as m
    return m


def dft_rows(n, rows, direction):
    """fp64 w_N^{b k} for the given b (exponent reduced exactly in int64)."""
    b = torch.as_tensor(rows, device="cuda", dtype=torch.int64)[:, None]
    k = torch.arange(n, device="cuda", dtype=torch.int64)[None, :]
    ph = ((b * k) % n).double() * (2 * math.pi / n) * (1.0 if direction > 0 else -1.0)
    return torch.complex(torch.cos(ph), torch.sin(ph))


def run_impulses(fg, n, rows, layout, direction, tuning=0, pass_radix=0):
    batch = len(rows)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, algorithm="stockham",
                                                 tuning=tuning, pass_radix=pass_radix))
    idx = torch.as_tensor(rows, device="cuda", dtype=torch.int64)
    if layout == "interleaved":
        x = torch.zeros(batch, n, 2, device="cuda")
        x[torch.arange(batch, device="cuda"), idx, 0] = 1.0
        y = torch.full_like(x, float("nan"))
        plan.execute(x, y, direction=direction)
        got = torch.view_as_complex(y)
    else:
        re = torch.zeros(batch, n, device="cuda")
        im = torch.zeros_like(re)
        re[torch.arange(batch, device="cuda"), idx] = 1.0
        ore, oim = torch.full_like(re, float("nan")), torch.full_like(im, float("nan"))
        plan.execute(re, ore, im, oim, direction=direction)
        got = torch.complex(ore, oim)
    torch.cuda.synchronize()
    return got


def max_err(got, want):
    return float((got.to(torch.complex128) - want).abs().max())


@pytest.mark.parametrize("l2", list(range(0, 15)))
@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
def test_full_dft_matrix_block_sizes(fg, l2, layout, direction):
    """N <= 2^14: all N impulses -> the complete N x N matrix (K2 kernels,
    TMA and direct variants)."""
    n = 1 << l2
    rows = list(range(n))
    chunk = max(1, (1 << 26) // n)  # bound the fp64 reference to 1 GiB
    for tuning in ((0, 1) if l2 >= 6 else (0,)):
        worst = 0.0
        for r0 in range(0, n, chunk):
            rs = rows[r0:r0 + chunk]
            got = run_impulses(fg, n, rs, layout, direction, tuning)
            worst = max(worst, max_err(got, dft_rows(n, rs, direction)))
            del got
        assert worst <= 2e-6, (n, layout, direction, tuning, worst)


@pytest.mark.parametrize("l2,hint", [(7, 8), (8, 8), (9, 8), (9, 16), (10, 8), (10, 16), (11, 8), (11, 16), (11, 32),
                                     (12, 8), (12, 16), (12, 32), (13, 16), (14, 16)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
@pytest.mark.parametrize("direction", [-1, 1])
def test_full_dft_matrix_radix_hint_plans(fg, l2, hint, layout, direction):
    """The radix hint's plans (register passes of radix <= 8 / 16 / 32 in the
    reference's Stockham shape, fftgen_config.pass_radix): complete matrix."""
    n = 1 << l2
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=1, pass_radix=hint))
    assert max(r for r, *_ in plan.passes()) <= hint and f"pass radix hint {hint}" in plan.describe()
    got = run_impulses(fg, n, list(range(n)), layout, direction, pass_radix=hint)
    assert max_err(got, dft_rows(n, list(range(n)), direction)) <= 2e-6


@pytest.mark.parametrize("l2,tuning", [(15, 0), (16, 0), (17, 0), (18, 0), (19, 0), (20, 0), (20, 1), (21, 0), (21, 8),
                                       (22, 0), (22, 16), (24, 0), (24, 16)])
@pytest.mark.parametrize("layout", ["interleaved", "split"])
def test_dft_matrix_rows_fourstep(fg, l2, tuning, layout):
    """K5 / K3 (two- and three-pass plans): full output rows for impulses at
    the ends, at powers of two and at random positions."""
    n = 1 << l2
    rng = np.random.default_rng(l2)
    nrows = 24 if l2 <= 20 else 8
    rows = sorted({0, 1, n // 2, n - 1, *(1 << rng.integers(0, l2, 4)).tolist(),
                   *rng.integers(0, n, nrows).tolist()})
    for direction in (-1, 1):
        got = run_impulses(fg, n, rows, layout, direction, tuning)
        assert max_err(got, dft_rows(n, rows, direction)) <= 2e-6, (n, tuning, layout, direction)
        del got


def test_cluster_and_unaligned_paths_same_matrix(fg):
    """2^15 through the K5 cluster kernel and through the two-launch path it
    falls back to for unaligned data: the same matrix rows."""
    n = 1 << 15
    rows = [0, 1, 3, 4097, n - 1]
    want = dft_rows(n, rows, -1)
    got = run_impulses(fg, n, rows, "interleaved", -1)
    assert max_err(got, want) <= 2e-6
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="interleaved", batch=len(rows), cluster_size=-1))
    x = torch.zeros(len(rows), n, 2, device="cuda")
    x[torch.arange(len(rows)), torch.as_tensor(rows), 0] = 1.0
    y = torch.empty_like(x)
    plan.execute(x, y)
    torch.cuda.synchronize()
    assert max_err(torch.view_as_complex(y), want) <= 2e-6
