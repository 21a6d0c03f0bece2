"""Multi-process paths on CPU (gloo, world size 2 and 4) and on one GPU (NCCL,
world size 1).

The CPU tests exercise the host logic of paper_2308_00497_b200.distributed --
batch shard ranges and the three all-to-all exchanges of the distributed
four-step -- with the pinned CPU oracle injected as the local FFT (product
code never imports the oracle), against the oracle's full transform.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_range_partitions_exactly():
    from paper_2308_00497_b200.distributed import shard_range
    for total in (0, 1, 7, 65536, 65537, 131071):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


# ---------------------------------------------------------------- gloo workers
def _oracle_fft(x: torch.Tensor, size: int, direction: int) -> torch.Tensor:
    """Test-side local FFT: the pinned oracle on a batch of complex rows."""
    orc = oracle.Oracle()
    inter = oracle.as_interleaved(x.numpy().astype(np.complex128))
    y = orc.forward(inter, "stockham", 4, inverse=direction > 0)
    return torch.from_numpy(oracle.as_complex(y).astype(np.complex64))


def _np_twiddle(blk: torch.Tensor, ro: int, co: int, n: int, direction: int) -> None:
    r = np.arange(blk.shape[0], dtype=np.int64)[:, None] + ro
    c = np.arange(blk.shape[1], dtype=np.int64)[None, :] + co
    e = (r * c) % n
    w = np.exp(direction * 2j * np.pi * e / n)
    blk.copy_(torch.from_numpy((blk.numpy().astype(np.complex128) * w).astype(np.complex64)))


def _dist_worker(rank, world, port, n, direction, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_00497_b200.distributed import DistributedFFT
        orc = oracle.Oracle()
        x = orc.seeded_input(n, 1).astype(np.float32).astype(np.float64)
        z = oracle.as_complex(x).astype(np.complex64)
        m = n // world
        d = DistributedFFT(n, local_fft=_oracle_fft, twiddle=_np_twiddle)
        local = torch.from_numpy(z[rank * m:(rank + 1) * m].copy())
        out = d.execute(local, direction=direction)
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        if rank == 0:
            q.put(torch.cat(gathered).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1 << 10), (4, 1 << 12), (2, 1 << 13)])
@pytest.mark.parametrize("direction", [-1, 1])
def test_distributed_four_step_gloo(world, n, direction):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, n, direction, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = oracle.Oracle()
    x = orc.seeded_input(n, 1).astype(np.float32).astype(np.float64)
    want = oracle.as_complex(orc.forward(x, "stockham", 4, inverse=direction > 0))
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-5 * np.log2(n), err


def test_distributed_rejects_bad_geometry():
    from paper_2308_00497_b200.distributed import DistributedFFT
    with pytest.raises(ValueError):
        DistributedFFT(1000)
    with pytest.raises(ValueError):
        DistributedFFT(1 << 10, n1=3)


# ---------------------------------------------------------------- one GPU, NCCL
def _nccl_single(n):
    from paper_2308_00497_b200.distributed import BatchShardedFFT, DistributedFFT
    import paper_2308_00497_b200 as fg
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.complex(torch.rand(n, device="cuda", generator=g) * 2 - 1,
                      torch.rand(n, device="cuda", generator=g) * 2 - 1)
    d = DistributedFFT(n)
    y = d.execute(x)
    plan = fg.compile_pipeline(fg.PipelineConfig(n=n, batch=1))
    ref = torch.empty_like(x)
    plan.execute(torch.view_as_real(x), torch.view_as_real(ref))
    torch.cuda.synchronize()
    rel = (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()
    back = d.execute(y, direction=fg.INVERSE) / n
    rt = (torch.linalg.norm(back - x) / torch.linalg.norm(x)).item()
    s = BatchShardedFFT(1024, 10, layout="interleaved")
    assert (s.start, s.count) == (0, 10)
    return rel, rt


@pytest.mark.gpu
@pytest.mark.parametrize("l2", [20, 24])
def test_distributed_four_step_nccl_world1(l2):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rel, rt = _nccl_single(1 << l2)
        assert rel < 5e-6 and rt < 1e-6, (rel, rt)
    finally:
        dist.destroy_process_group()
