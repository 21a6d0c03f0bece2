"""The four-step twiddle tables the K3 / K5 kernels read (generated on the
device by K4, fp64 sincospi of an exact argument) against the reference's
unit_root formula (matrix.cpp:14-35) rounded once to fp32.

Entry e of a table is w_s^t, t = its exponent; both sides reduce t exactly in
integers and are exact at quadrant multiples.  The two fp64 evaluations
(device sincospi vs host cos/sin) may differ in their last fp64 bits, which
survives the fp32 rounding only when a value lies within an fp64 ulp of an
fp32 rounding boundary: the test asserts bitwise equality except for at most
1e-6 of the entries, and never more than 1 fp32 ulp.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    assert torch.cuda.is_available()
    import paper_2308_00497_b200 as m
    return m


def unit_root_f32(s, t):
    t = np.asarray(t, dtype=np.int64) % s
    ang = -2.0 * np.pi * t.astype(np.float64) / float(s)
    re, im = np.cos(ang), np.sin(ang)
    quad = (4 * t) % s == 0
    q = (4 * t // s) % 4
    re = np.where(quad, np.array([1.0, 0.0, -1.0, 0.0])[q], re)
    im = np.where(quad, np.array([0.0, -1.0, 0.0, 1.0])[q], im)
    return (re.astype(np.float32) + 1j * im.astype(np.float32)).astype(np.complex64), quad


def compare(got, want, quad):
    assert got.shape == want.shape
    g = got.view(np.float32).reshape(-1, 2)
    w = want.view(np.float32).reshape(-1, 2)
    same = np.all(g == w, axis=1)
    assert np.all(same[quad]), "quadrant entries must be exact"
    diff = np.abs(g - w)
    ulp = np.spacing(np.abs(w).astype(np.float32))
    assert np.all(diff <= ulp + 1e-45), float(np.max(diff / np.maximum(ulp, 1e-45)))
    assert (~same).sum() <= max(1, int(1e-6 * same.size)), int((~same).sum())


@pytest.mark.parametrize("l2", [15, 16, 18, 21, 24, 28])
def test_group_tables_are_unit_root_in_fp32(fg, l2):
    n = 1 << l2
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout="interleaved", batch=1, algorithm="stockham",
                                                 cluster_size=-1))
    groups = plan.passes()  # (NS, cols, k, s) per group
    checked = 0
    for g, (ns, cols, k, s) in enumerate(groups):
        q = plan.group_twiddles(g, 0)
        p = plan.group_twiddles(g, 1)
        if cols == 1:
            assert q.size == 0 and p.size == 0
            continue
        r0 = q.size // cols
        assert q.size == r0 * cols and p.size == (ns // r0) * cols
        # Q[A0][m] = w_s^{A0 (NS/R0) m}
        a0 = np.arange(r0, dtype=np.int64)[:, None]
        m = np.arange(cols, dtype=np.int64)[None, :]
        want, quad = unit_root_f32(s, a0 * (ns // r0) * m)
        compare(q, want.reshape(-1), quad.reshape(-1))
        # P = w_s^{c m}: [c][m] for column groups, [m][c] for the rows group (k == 1)
        c = np.arange(ns // r0, dtype=np.int64)
        e = (m.T * c[None, :]) if k == 1 else (c[:, None] * m)
        want, quad = unit_root_f32(s, e)
        compare(p, want.reshape(-1), quad.reshape(-1))
        checked += 1
    assert checked == len(groups) - 1
