"""Multi-process paths on CPU: gloo at world size 2 and 4, plus an in-process
emulation of P = 1..16 ranks.

They exercise the host logic of paper_2308_00497_b200.distributed -- batch
shard ranges and the three contiguous-chunk all-to-alls of the distributed
four-step -- with a numpy restatement of the three per-rank stages (the local
transform by the pinned oracle; product code never imports the oracle),
against the oracle's full transform.  The same composition with the sm_100a
stages runs on one GPU in tests/test_gpu_distributed.py.
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


# ------------------------------------------------- numpy restatement of the stages
class NumpyStages:
    """Test-side restatement of the three per-rank stages of csrc/dist.cu on
    CPU complex64 tensors (the butterfly's P-point DFT and w_N twiddle in fp64,
    the local M-point transform by the pinned oracle)."""

    def __init__(self, n, world, rank):
        self.n, self.P, self.q = n, world, rank
        self.m = n // world
        self.l1 = self.m // world

    def butterfly(self, recv, send, direction):
        P, l1, n = self.P, self.l1, self.n
        r1 = recv.numpy().astype(np.complex128).reshape(P, l1)
        sgn = 1.0 if direction > 0 else -1.0
        kb = np.arange(P)
        dftP = np.exp(sgn * 2j * np.pi * np.outer(kb, kb) / P)          # [k_b][r]
        y = dftP @ r1                                                     # [k_b][j]
        a = self.q * l1 + np.arange(l1)
        y *= np.exp(sgn * 2j * np.pi * ((np.outer(kb, a)) % n) / n)
        send.copy_(torch.from_numpy(y.reshape(-1).astype(np.complex64)))

    def local(self, inp, out, direction):
        orc = oracle.Oracle()
        inter = oracle.as_interleaved(inp.numpy().astype(np.complex128)[None, :])
        y = orc.forward(inter, "stockham", 4, inverse=direction > 0)
        out.copy_(torch.from_numpy(oracle.as_complex(y)[0].astype(np.complex64)))

    def unpack(self, recv, out):
        out.copy_(recv.reshape(self.P, self.l1).t().reshape(-1))


def _want(n, direction):
    orc = oracle.Oracle()
    x = orc.seeded_input(n, 1).astype(np.float32).astype(np.float64)
    z = oracle.as_complex(x).astype(np.complex64)
    want = oracle.as_complex(orc.forward(x, "stockham", 4, inverse=direction > 0))
    return z, want


@pytest.mark.parametrize("world,n", [(1, 1 << 8), (2, 1 << 10), (4, 1 << 12), (8, 1 << 12), (16, 1 << 12)])
@pytest.mark.parametrize("direction", [-1, 1])
def test_emulated_composition_numpy_stages(world, n, direction):
    """The exchange pattern + stage algebra of the distributed four-step, all
    P ranks in one process (emulated_exchange), against the oracle."""
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    z, want = _want(n, direction)
    e = EmulatedDistributedFFT(n, world, stages_factory=lambda r: NumpyStages(n, world, r))
    m = n // world
    outs = e.execute([torch.from_numpy(z[r * m:(r + 1) * m].copy()) for r in range(world)], direction)
    got = torch.cat(outs).numpy()
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-5 * np.log2(n), err


@pytest.mark.parametrize("world,n", [(2, 1 << 10), (4, 1 << 12), (8, 1 << 12)])
def test_emulated_cyclic_output_order(world, n):
    """output_order="cyclic": rank s ends with X[s + P j] after two exchanges."""
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    z, want = _want(n, -1)
    e = EmulatedDistributedFFT(n, world, stages_factory=lambda r: NumpyStages(n, world, r), output_order="cyclic")
    m = n // world
    outs = e.execute([torch.from_numpy(z[r * m:(r + 1) * m].copy()) for r in range(world)], -1)
    got = np.empty(n, dtype=np.complex128)
    for s in range(world):
        got[s::world] = outs[s].numpy()
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-5 * np.log2(n), err
    with pytest.raises(ValueError):
        EmulatedDistributedFFT(n, world, stages_factory=lambda r: NumpyStages(n, world, r), output_order="bitrev")


# ---------------------------------------------------------------- gloo workers
def _dist_worker(rank, world, port, n, direction, q, order="natural"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_00497_b200.distributed import DistributedFFT
        z, _ = _want(n, direction)
        m = n // world
        d = DistributedFFT(n, stages=NumpyStages(n, world, rank), output_order=order)
        local = torch.from_numpy(z[rank * m:(rank + 1) * m].copy())
        out = d.execute(local, direction=direction)
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        if rank == 0:
            if order == "cyclic":  # rank s holds X[s + P j]
                full = np.empty(n, dtype=np.complex128)
                for s_, g in enumerate(gathered):
                    full[s_::world] = g.numpy()
                q.put(full)
            else:
                q.put(torch.cat(gathered).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,order", [(2, 1 << 10, "natural"), (4, 1 << 12, "natural"), (2, 1 << 13, "natural"),
                                           (2, 1 << 10, "cyclic")])
@pytest.mark.parametrize("direction", [-1, 1])
def test_distributed_four_step_gloo(world, n, order, direction):
    """Real process group (gloo all_to_all_single), world 2 / 4; both output orders."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, n, direction, q, order)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, want = _want(n, direction)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-5 * np.log2(n), err


def test_distributed_rejects_bad_geometry():
    from paper_2308_00497_b200.distributed import DistributedFFT, EmulatedDistributedFFT
    with pytest.raises(ValueError):
        DistributedFFT(1000, world=1, rank=0, stages=object())
    with pytest.raises(ValueError):
        EmulatedDistributedFFT(1 << 10, 3, stages_factory=lambda r: None)
    with pytest.raises(ValueError):
        EmulatedDistributedFFT(64, 8, stages_factory=lambda r: None)   # n < 2 world^2
