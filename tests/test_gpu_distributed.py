"""GPU parity of the distributed four-step (config C5, csrc/dist.cu +
paper_2308_00497_b200/distributed.py) with the real sm_100a stages.

P ranks are emulated on ONE device (EmulatedDistributedFFT: the per-rank
butterfly / local / unpack kernels with each rank's own twiddle offset, the
three all-to-alls as device copies of the same contiguous chunks NCCL would
move), and the one-rank NCCL path runs through torch.distributed for real.
Reference: the pinned fp64 oracle on fp32-rounded seeded inputs (relative L2
<= 1e-5 log2 N), and single tones where the oracle is too slow.
Each stage is also checked on its own against an fp64 numpy restatement.
"""
import ctypes
import math
import os
import socket

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


def seeded_complex(orc, n, seed=1):
    x = orc.seeded_input(n, seed).astype(np.float32).astype(np.float64)
    return x, oracle.as_complex(x).astype(np.complex64)


def blocks_of(z, world):
    m = z.size // world
    return [torch.from_numpy(z[r * m:(r + 1) * m].copy()).cuda() for r in range(world)]


# ------------------------------------------------------------- single stages
@pytest.mark.parametrize("world", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("direction", [-1, 1])
def test_butterfly_stage_vs_fp64(fg, world, direction):
    n = 1 << 16
    rank = world - 1
    p = fg.DistPlan(n, world, rank)
    g = torch.Generator(device="cuda").manual_seed(world)
    recv = torch.complex(torch.rand(p.block, device="cuda", generator=g) - .5,
                         torch.rand(p.block, device="cuda", generator=g) - .5)
    send = torch.full_like(recv, float("nan"))
    p.butterfly(recv, send, direction)
    torch.cuda.synchronize()
    l1 = p.chunk
    r1 = recv.cpu().numpy().astype(np.complex128).reshape(world, l1)
    sgn = 1.0 if direction > 0 else -1.0
    kb = np.arange(world)
    y = np.exp(sgn * 2j * np.pi * np.outer(kb, kb) / world) @ r1
    a = rank * l1 + np.arange(l1)
    y *= np.exp(sgn * 2j * np.pi * (np.outer(kb, a) % n) / n)
    got = send.cpu().numpy().reshape(world, l1)
    assert np.linalg.norm(got - y) / np.linalg.norm(y) < 3e-7


@pytest.mark.parametrize("world", [1, 2, 4, 8, 16])
def test_unpack_stage_is_the_stride_world_interleave(fg, world):
    n = 1 << 14
    p = fg.DistPlan(n, world, 0)
    src = torch.arange(p.block, device="cuda", dtype=torch.float32).to(torch.complex64)
    out = torch.empty_like(src)
    p.unpack(src, out)
    torch.cuda.synchronize()
    assert torch.equal(out, src.reshape(world, p.chunk).t().reshape(-1))


def test_dist_plan_validation(fg):
    with pytest.raises(fg.PlanError):
        fg.DistPlan(3000, 2, 0)
    with pytest.raises(fg.DimensionError):
        fg.DistPlan(1 << 10, 3, 0)
    with pytest.raises(fg.DimensionError):
        fg.DistPlan(1 << 10, 4, 4)
    with pytest.raises(fg.DimensionError):
        fg.DistPlan(16, 4, 0)
    p = fg.DistPlan(1 << 12, 2, 1)
    x = torch.zeros(p.block, dtype=torch.complex64, device="cuda")
    with pytest.raises(fg.ExecError):
        p.butterfly(x, x)                                   # out of place only
    with pytest.raises(fg.DimensionError):
        p.unpack(x, torch.zeros(p.block + 2, dtype=torch.complex64, device="cuda"))
    assert "kernel" in p.describe_local() and p.local_launches() >= 1


# ------------------------------------------------ emulated ranks vs the oracle
@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("direction", [-1, 1])
def test_emulated_2p20_vs_oracle(fg, orc, world, direction):
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n = 1 << 20
    x, z = seeded_complex(orc, n)
    e = EmulatedDistributedFFT(n, world)
    got = torch.cat(e.execute(blocks_of(z, world), direction)).cpu().numpy()
    want = oracle.as_complex(orc.forward(x[None], "stockham", 4, inverse=direction > 0, threads=4))[0]
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err <= tol(n) and err < 3e-6, err


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_emulated_cyclic_output_order(fg, orc, world, transport):
    """output_order="cyclic" (two exchanges): rank s holds X[s + P j], the
    same values the natural-order path unpacks, bitwise."""
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n = 1 << 20
    x, z = seeded_complex(orc, n)
    blocks = blocks_of(z, world)
    cyc = EmulatedDistributedFFT(n, world, transport=transport, output_order="cyclic").execute(blocks)
    nat = torch.cat(EmulatedDistributedFFT(n, world, transport=transport).execute(blocks))
    got = torch.empty_like(nat)
    for s in range(world):
        got[s::world] = cyc[s]
    assert torch.equal(got, nat)
    want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=4))[0]
    err = np.linalg.norm(got.cpu().numpy() - want) / np.linalg.norm(want)
    assert err <= tol(n), err


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_2p24_vs_oracle(fg, orc, world):
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n = 1 << 24
    x, z = seeded_complex(orc, n, seed=3)
    e = EmulatedDistributedFFT(n, world)
    got = torch.cat(e.execute(blocks_of(z, world))).cpu().numpy()
    want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=8))[0]
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err <= tol(n) and err < 4e-6, err


def tone_blocks(n, world, k0, direction=1):
    """x[t] = exp(direction * 2 pi i k0 t / N), exact phase reduction in int64."""
    m = n // world
    out = []
    for r in range(world):
        t = torch.arange(r * m, (r + 1) * m, device="cuda", dtype=torch.int64)
        ph = ((t * k0) % n).double() * (2 * math.pi / n) * direction
        out.append(torch.complex(torch.cos(ph).float(), torch.sin(ph).float()))
        del t, ph
    return out


@pytest.mark.parametrize("world,l2", [(4, 30), (8, 28), (2, 26)])
def test_emulated_large_single_tone(fg, world, l2):
    """C5 sizes: forward of a tone exp(+2 pi i k0 t / N) is N delta[k - k0]."""
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n = 1 << l2
    k0 = 123457 % n
    e = EmulatedDistributedFFT(n, world)
    outs = e.execute(tone_blocks(n, world, k0))
    m = n // world
    err2 = 0.0
    for r, o in enumerate(outs):
        o = o.to(torch.complex128)
        if r * m <= k0 < (r + 1) * m:
            o[k0 - r * m] -= n
        err2 += float(torch.sum(o.real ** 2 + o.imag ** 2))
        del o
    rel = math.sqrt(err2) / n
    assert rel < tol(n), rel


def test_emulated_round_trip_2p22(fg, orc):
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n, world = 1 << 22, 4
    _, z = seeded_complex(orc, n, seed=9)
    e = EmulatedDistributedFFT(n, world)
    back = e.execute(e.execute(blocks_of(z, world), -1), 1)
    got = torch.cat(back).cpu().numpy() / n
    assert np.linalg.norm(got - z) / np.linalg.norm(z) < 1e-6


# ------------------------------------- peer-memory transport (fused exchanges)
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_p2p_bitwise_equals_nccl_path(fg, orc, world):
    """The peer-pointer kernels (exchanges as loads / stores inside the
    butterfly and unpack) compute exactly what the contiguous-chunk NCCL
    pipeline computes: same arithmetic, other addresses -> bitwise equal."""
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n = 1 << 20
    x, z = seeded_complex(orc, n, seed=6)
    blocks = blocks_of(z, world)
    a = torch.cat(EmulatedDistributedFFT(n, world).execute(blocks))
    b = torch.cat(EmulatedDistributedFFT(n, world, transport="p2p").execute(blocks))
    assert torch.equal(a, b)
    want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=4))[0]
    got = b.cpu().numpy()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 3e-6


def test_emulated_p2p_2p30_tone(fg):
    """C5 size through the fused peer kernels: the inverse of the tone
    exp(+2 pi i k0 t / N) is N delta[k + k0 mod N]."""
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n, world, k0 = 1 << 30, 4, 987654
    outs = EmulatedDistributedFFT(n, world, transport="p2p").execute(tone_blocks(n, world, k0), 1)
    m, peak = n // world, (-k0) % n
    err2 = 0.0
    for r, o in enumerate(outs):
        o = o.to(torch.complex128)
        if r * m <= peak < (r + 1) * m:
            o[peak - r * m] -= n
        err2 += float(torch.sum(o.real ** 2 + o.imag ** 2))
        del o
    assert math.sqrt(err2) / n < tol(n)


def test_peer_tables_validated(fg):
    p = fg.DistPlan(1 << 12, 2, 0)
    x = torch.zeros(p.block, dtype=torch.complex64, device="cuda")
    y = torch.zeros_like(x)
    with pytest.raises(fg.DimensionError):
        p.butterfly_peers([x], [y])
    with pytest.raises(fg.ExecError):
        p.butterfly_peers([x, 0], [y, y])
    with pytest.raises(fg.ExecError):
        p.unpack_peers([x, y], y)                  # out aliases a source block
    with pytest.raises(fg.ExecError):
        p.butterfly_peers([x, y], [y, torch.zeros_like(x)])   # a receive block is an input block


def test_distributed_p2p_symmetric_memory_world1(fg, orc):
    """transport='p2p' under a real process group: torch symmetric memory
    rendezvous, device barriers, the fused kernels (world 1 on this box)."""
    import torch.distributed as dist
    from paper_2308_00497_b200.distributed import DistributedFFT
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1 << 22
        try:
            d = DistributedFFT(n, transport="p2p")
        except Exception as e:  # symmetric memory unavailable in this configuration
            pytest.skip(f"symmetric memory rendezvous failed: {e}")
        x, z = seeded_complex(orc, n, seed=8)
        d.input_block().copy_(torch.from_numpy(z).cuda())
        got = d.execute(d.input_block()).cpu().numpy()
        want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=8))[0]
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 4e-6
    finally:
        dist.destroy_process_group()


# ----------------------------------------------------- one rank, real NCCL
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("l2", [20, 24])
def test_distributed_nccl_world1_vs_oracle(fg, orc, l2):
    """DistributedFFT under a real NCCL process group (world 1): the same
    butterfly / local / unpack stages, exchanges through all_to_all_single's
    world-1 path; no shortcut to the single-GPU plan."""
    import torch.distributed as dist
    from paper_2308_00497_b200.distributed import DistributedFFT
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1 << l2
        x, z = seeded_complex(orc, n, seed=2)
        d = DistributedFFT(n)
        got = d.execute(torch.from_numpy(z).cuda()).cpu().numpy()
        want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=8))[0]
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= tol(n) and err < 4e-6, err
    finally:
        dist.destroy_process_group()


def test_dist_execute_with_exchange_callback(fg, orc):
    """fftgen_dist_execute (the C-ABI pipeline a C++/NCCL host calls) with an
    exchange callback; world 1, where the all-to-all is a device copy."""
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_void_p]
    calls = []

    @ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                      ctypes.c_void_p)
    def exchange(ctx, send, recv, chunk_bytes, stream):
        calls.append(chunk_bytes)
        return cudart.cudaMemcpyAsync(recv, send, chunk_bytes, 3, stream)

    n = 1 << 18
    x, z = seeded_complex(orc, n, seed=4)
    p = fg.DistPlan(n, 1, 0)
    src = torch.from_numpy(z).cuda()
    out, w0, w1 = (torch.empty_like(src) for _ in range(3))
    stream = torch.cuda.current_stream().cuda_stream
    fg._check(fg.lib.fftgen_dist_execute(p._h, -1, src.data_ptr(), out.data_ptr(), w0.data_ptr(), w1.data_ptr(),
                                         ctypes.cast(exchange, ctypes.c_void_p), None, stream))
    torch.cuda.synchronize()
    assert calls == [8 * n] * 3
    want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=4))[0]
    got = out.cpu().numpy()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 3e-6


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cyclic", [False, True])
def test_dist_execute_c_abi_ranks_in_threads(fg, orc, world, cyclic):
    """fftgen_dist_execute / _execute_cyclic with `world` ranks, one host
    thread each, all on this GPU: the exchange callback is a real all-to-all
    (a barrier, then rank r pulls chunk r of every rank's send buffer; one
    in-order stream orders the copies after every rank's producer kernel)."""
    import threading
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_void_p]
    n = 1 << 18
    m = n // world
    x, z = seeded_complex(orc, n, seed=6)
    plans = [fg.DistPlan(n, world, r) for r in range(world)]
    zs = torch.from_numpy(z).cuda()
    blocks = [zs[r * m:(r + 1) * m].clone() for r in range(world)]
    outs, w0s, w1s = ([torch.empty_like(b) for b in blocks] for _ in range(3))
    torch.cuda.synchronize()
    sends = [0] * world
    bar = threading.Barrier(world)
    calls = [0] * world

    def make_exchange(r):
        @ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                          ctypes.c_void_p)
        def exchange(ctx, send, recv, chunk_bytes, stream):
            calls[r] += 1
            sends[r] = send
            bar.wait()
            for q in range(world):
                if cudart.cudaMemcpyAsync(recv + q * chunk_bytes, sends[q] + r * chunk_bytes, chunk_bytes, 3,
                                          stream):
                    return 1
            bar.wait()
            return 0
        return exchange

    cbs = [make_exchange(r) for r in range(world)]
    fn = fg.lib.fftgen_dist_execute_cyclic if cyclic else fg.lib.fftgen_dist_execute
    status = [None] * world

    def run(r):
        status[r] = fn(plans[r]._h, -1, blocks[r].data_ptr(), outs[r].data_ptr(), w0s[r].data_ptr(),
                       w1s[r].data_ptr(), ctypes.cast(cbs[r], ctypes.c_void_p), None, None)

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=120)
    torch.cuda.synchronize()
    assert status == [0] * world and calls == [2 if cyclic else 3] * world
    if cyclic:
        got = torch.empty_like(zs)
        for s in range(world):
            got[s::world] = outs[s]
    else:
        got = torch.cat(outs)
    want = oracle.as_complex(orc.forward(x[None], "stockham", 4, threads=4))[0]
    err = np.linalg.norm(got.cpu().numpy() - want) / np.linalg.norm(want)
    assert err <= tol(n) and err < 3e-6, err
    # bitwise the emulated pipeline (same kernels, same chunks)
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    e = EmulatedDistributedFFT(n, world, output_order="cyclic" if cyclic else "natural").execute(blocks)
    assert all(torch.equal(a, b) for a, b in zip(e, outs))


# ----------------------------------------------- fftgen_twiddle_multiply
@pytest.mark.parametrize("direction", [-1, 1])
@pytest.mark.parametrize("rows,cols,ro,co,n", [(64, 96, 3, 17, 1 << 20), (37, 33, 1000, 5, 1 << 30),
                                               (16, 512, 0, 0, 4096), (8, 8, 123, 456, 777)])
def test_twiddle_multiply_vs_fp64(fg, direction, rows, cols, ro, co, n):
    g = torch.Generator(device="cuda").manual_seed(rows)
    full = torch.complex(torch.rand(rows, cols + 7, device="cuda", generator=g),
                         torch.rand(rows, cols + 7, device="cuda", generator=g))
    blk = full[:, :cols]                                      # ld = cols + 7
    before = full.clone()
    fg.twiddle_multiply(blk, ro, co, n, direction)
    torch.cuda.synchronize()
    r = np.arange(rows, dtype=np.int64)[:, None] + ro
    c = np.arange(cols, dtype=np.int64)[None, :] + co
    w = np.exp((1.0 if direction > 0 else -1.0) * 2j * np.pi * ((r * c) % n) / n)
    want = before[:, :cols].cpu().numpy().astype(np.complex128) * w
    got = full[:, :cols].cpu().numpy()
    assert np.max(np.abs(got - want)) < 4e-7 * np.max(np.abs(want))
    assert torch.equal(full[:, cols:], before[:, cols:])     # the padding is untouched
    # quadrant exponents are exact: w = 1, -i, -1, +i
    q = torch.ones(1, 4, dtype=torch.complex64, device="cuda")
    fg.twiddle_multiply(q, 1, 0, 4, -1)
    torch.cuda.synchronize()
    assert torch.equal(q.cpu(), torch.tensor([[1, -1j, -1, 1j]], dtype=torch.complex64))
