"""Multi-GPU partitioning of the FFT hot path, one process per GPU.

* BatchShardedFFT -- batched transforms (configs C2/C3) shard by contiguous
  batch ranges; every rank owns its own plan and twiddle tables and there is
  NO data-path collective (weak scaling).
* DistributedFFT  -- one very large transform (config C5, N = 2^30) block
  distributed over P ranks (rank r holds x[r M : (r+1) M], M = N/P).  The
  reference's two-factor split (formula.cpp:160-165, Eq. 1) with K = P:

    X[k_b + P k_a] = sum_a w_M^{a k_a} (w_N^{a k_b} sum_r x[a + M r] w_P^{r k_b})

  runs as three all-to-alls of CONTIGUOUS equal chunks (NCCL grouped
  send/recv through torch.distributed.all_to_all_single; no pack or
  transpose copy on either side) around three sm_100a stages of the C ABI
  (fftgen_dist_*, csrc/dist.cu):

    1. exchange   the input block as-is            -> R1[r][j] = x[r M + q L1 + j]
    2. butterfly  P-point DFT over r + D^N twiddle, stored per destination rank
    3. exchange                                    -> R2 = the natural M-point input
    4. local      the single-GPU M-point plan (K2 / K5 / K3)
    5. exchange   contiguous output chunks         -> R3[q'][j] = X[s M + P j + q']
    6. unpack     out[P j + q'] = R3[q'][j]  (the stride-P interleave of Pi^N_P)

  L1 = N/P^2.  output_order="cyclic" (the transposed-order output of SURVEY
  8e) stops after step 4: rank s then holds X[s + P j], j < M -- the cyclic
  distribution -- and the third all-to-all and the unpack are skipped (two
  exchanges instead of three; a consumer that transforms back, e.g. a
  convolution, takes the same order).  The stages are injectable so the exchange logic is testable on
  CPU with gloo (tests/test_distributed.py, a numpy restatement of the three
  stages) and `EmulatedDistributedFFT` runs P ranks in lockstep on ONE GPU
  with the real kernels, the exchanges being device copies of the same
  chunks (tests/test_gpu_distributed.py).

  transport="p2p" runs the same algebra with the exchanges INSIDE the
  kernels over peer memory (torch symmetric memory: every rank's blocks are
  mapped into every process over NVLink): the butterfly pulls chunk q of
  every rank's input and pushes row k_b into rank k_b's receive block
  (exchanges 1 and 2), the local plan runs on the rank's own block, and the
  unpack pulls slot q of every rank's result (exchange 3) -- three kernels
  (+ the local plan) and four device barriers, no NCCL kernels or staging
  copies.
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch
import torch.distributed as dist

from . import FORWARD, DistPlan, PipelineConfig, compile_pipeline


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, start+count) batch range of `rank`; ranks differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, rem = divmod(total, world)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


def _rank_world(group) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


class BatchShardedFFT:
    """This rank's share of a batched FFT; no communication on the data path."""

    def __init__(self, n: int, global_batch: int, layout: str = "split", device: Optional[int] = None,
                 group=None, rank: Optional[int] = None, world: Optional[int] = None):
        r, w = _rank_world(group)
        self.rank = r if rank is None else rank
        self.world = w if world is None else world
        self.start, self.count = shard_range(global_batch, self.rank, self.world)
        if device is None:
            device = torch.cuda.current_device()
        self.plan = compile_pipeline(PipelineConfig(n=n, layout=layout, batch=max(self.count, 1),
                                                    device=device, algorithm="stockham"))

    def execute(self, in0, out0, in1=None, out1=None, direction: int = FORWARD, stream=None) -> None:
        """Tensors hold this rank's `count` transforms (the local shard)."""
        if self.count:
            self.plan.execute(in0, out0, in1, out1, direction=direction, stream=stream)


ORDERS = ("natural", "cyclic")


def _check_order(order: str) -> str:
    if order not in ORDERS:
        raise ValueError(f"output_order must be 'natural' or 'cyclic', got {order!r}")
    return order


def check_geometry(n: int, world: int) -> None:
    if n < 4 or n & (n - 1):
        raise ValueError(f"n must be a power of two >= 4, got {n}")
    if world not in (1, 2, 4, 8, 16):
        raise ValueError(f"world size must be 1, 2, 4, 8 or 16, got {world}")
    if n < 2 * world * world:
        raise ValueError(f"n = {n} is below 2 * world^2 = {2 * world * world}")


class DistributedFFT:
    """One N-point transform block-distributed over the process group.

    `stages` supplies butterfly(recv, send, direction), local(inp, out,
    direction) and unpack(recv, out) on this rank's blocks; the default is the
    sm_100a DistPlan.  `exchange(send, recv)` defaults to
    all_to_all_single over the group (a copy when the world is 1).
    transport="p2p" fuses the exchanges into the kernels over symmetric
    (peer-mapped) memory instead; `input_block()` is then the zero-copy
    input buffer.  output_order="cyclic" returns X[rank + P j] (j < M)
    without the third exchange."""

    def __init__(self, n: int, group=None, device: Optional[int] = None, rank: Optional[int] = None,
                 world: Optional[int] = None, stages=None, transport: str = "nccl", output_order: str = "natural"):
        r, w = _rank_world(group)
        self.group = group
        self.rank = r if rank is None else rank
        self.world = w if world is None else world
        check_geometry(n, self.world)
        self.n = n
        self.m = n // self.world
        self.l1 = self.m // self.world
        self.output_order = _check_order(output_order)
        if stages is None:
            if device is None:
                device = torch.cuda.current_device()
            stages = DistPlan(n, self.world, self.rank, device)
        self.stages = stages
        self._work: dict = {}
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport must be 'nccl' or 'p2p', got {transport!r}")
        self.transport = transport
        self._symm = None
        if transport == "p2p":
            self._init_symmetric(device if device is not None else torch.cuda.current_device())

    # ---- peer-memory transport ----------------------------------------------
    def _init_symmetric(self, device: int) -> None:
        """One symmetric allocation [input | receive | local result] per rank,
        rendezvoused over the group: every rank's blocks become addressable
        here (NVLink peer mappings)."""
        import torch.distributed._symmetric_memory as symm_mem
        m = self.m
        buf = symm_mem.empty(3 * m, dtype=torch.complex64, device=torch.device("cuda", device))
        group = self.group if self.group is not None else dist.group.WORLD
        handle = symm_mem.rendezvous(buf, group)
        ptrs = [int(p) for p in handle.buffer_ptrs]
        self._symm = (buf, handle)
        self._blocks = buf.view(3, m)
        self._peer = {name: [p + i * 8 * m for p in ptrs] for i, name in enumerate(("x", "recv", "z"))}

    def input_block(self) -> torch.Tensor:
        """p2p: this rank's input block in symmetric memory (fill it, then call
        execute(input_block()) to skip the copy-in)."""
        if self._symm is None:
            raise RuntimeError("input_block() needs transport='p2p'")
        return self._blocks[0]

    def _barrier(self) -> None:
        self._symm[1].barrier()

    def _execute_p2p(self, x_local: torch.Tensor, direction: int, out: torch.Tensor) -> torch.Tensor:
        x_blk, recv_blk, z_blk = self._blocks[0], self._blocks[1], self._blocks[2]
        if x_local.data_ptr() != x_blk.data_ptr():
            x_blk.copy_(x_local)
        self._barrier()                       # every rank's input is in place
        self.stages.butterfly_peers(self._peer["x"], self._peer["recv"], direction)
        self._barrier()                       # every receive block is complete
        if self.output_order == "cyclic":     # X[rank + P j]: no third exchange
            self.stages.local(recv_blk, out, direction)
            return out                        # the next execute's first barrier orders the reuse
        self.stages.local(recv_blk, z_blk, direction)
        self._barrier()                       # every local result is complete
        self.stages.unpack_peers(self._peer["z"], out)
        self._barrier()                       # no rank still reads this rank's blocks
        return out

    def exchange(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        """All-to-all of `world` contiguous chunks: send chunk q -> rank q, recv chunk r <- rank r."""
        if self.world == 1 and not (dist.is_available() and dist.is_initialized()):
            recv.copy_(send)
        else:
            dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), group=self.group)

    def workspace(self, like: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        key = (like.device, like.dtype)
        if key not in self._work:
            self._work[key] = (torch.empty(self.m, dtype=like.dtype, device=like.device),
                               torch.empty(self.m, dtype=like.dtype, device=like.device))
        return self._work[key]

    def execute(self, x_local: torch.Tensor, direction: int = FORWARD,
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """x_local: complex64 (M,) = x[rank*M : (rank+1)*M]; returns X^ of the same
        block (output_order "cyclic": X^[rank + P j], j < M)."""
        if x_local.numel() != self.m or x_local.dtype != torch.complex64:
            raise ValueError(f"expected a complex64 block of {self.m} elements")
        x_local = x_local.reshape(-1)
        if out is None:
            out = torch.empty_like(x_local)
        if self.world == 1 and self.transport == "nccl":
            # P = 1: both exchanges, the 1-point butterfly (w^0 = 1) and the
            # stride-1 unpack are identities; the local plan is the transform
            self.stages.local(x_local, out, direction)
            return out
        if self.transport == "p2p":
            return self._execute_p2p(x_local, direction, out)
        w0, w1 = self.workspace(x_local)
        self.exchange(x_local, w0)
        self.stages.butterfly(w0, w1, direction)
        self.exchange(w1, w0)
        if self.output_order == "cyclic":
            self.stages.local(w0, out, direction)
            return out
        self.stages.local(w0, w1, direction)
        self.exchange(w1, w0)
        self.stages.unpack(w0, out)
        return out


def emulated_exchange(sends: Sequence[torch.Tensor], recvs: Sequence[torch.Tensor], chunk: int) -> None:
    """The all-to-all of P ranks held by one process: chunk q of rank r's send
    buffer lands as chunk r of rank q's receive buffer (what NCCL moves)."""
    P = len(sends)
    for r in range(P):
        for q in range(P):
            recvs[q][r * chunk:(r + 1) * chunk].copy_(sends[r][q * chunk:(q + 1) * chunk])


class EmulatedDistributedFFT:
    """P ranks of the distributed four-step in lockstep on one device: the
    real per-rank stages (kernels, twiddle offsets, chunk layouts), with the
    three all-to-alls as device copies.  Tests the composition the NCCL path
    runs, on one GPU."""

    def __init__(self, n: int, world: int, device: Optional[int] = None, stages_factory=None,
                 transport: str = "nccl", output_order: str = "natural"):
        check_geometry(n, world)
        self.output_order = _check_order(output_order)
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport must be 'nccl' or 'p2p', got {transport!r}")
        self.transport = transport
        self.n, self.world = n, world
        self.m = n // world
        self.l1 = self.m // world
        if stages_factory is None:
            dev = torch.cuda.current_device() if device is None else device
            stages_factory = lambda r: DistPlan(n, world, r, dev)  # noqa: E731
        self.stages = [stages_factory(r) for r in range(world)]

    def execute(self, blocks: Sequence[torch.Tensor], direction: int = FORWARD) -> list[torch.Tensor]:
        P = self.world
        if len(blocks) != P or any(b.numel() != self.m or b.dtype != torch.complex64 for b in blocks):
            raise ValueError(f"expected {P} complex64 blocks of {self.m} elements")
        blocks = [b.reshape(-1) for b in blocks]
        w0 = [torch.empty_like(b) for b in blocks]
        w1 = [torch.empty_like(b) for b in blocks]
        out = [torch.empty_like(b) for b in blocks]
        if self.transport == "p2p":
            # the same peer-pointer kernels the multi-process path runs; stream
            # order on one device stands in for the barriers between stages
            for r in range(P):
                self.stages[r].butterfly_peers(blocks, w0, direction)
            if self.output_order == "cyclic":
                for r in range(P):
                    self.stages[r].local(w0[r], out[r], direction)
                return out
            for r in range(P):
                self.stages[r].local(w0[r], w1[r], direction)
            for r in range(P):
                self.stages[r].unpack_peers(w1, out[r])
            return out
        emulated_exchange(blocks, w0, self.l1)
        for r in range(P):
            self.stages[r].butterfly(w0[r], w1[r], direction)
        emulated_exchange(w1, w0, self.l1)
        if self.output_order == "cyclic":
            for r in range(P):
                self.stages[r].local(w0[r], out[r], direction)
            return out
        for r in range(P):
            self.stages[r].local(w0[r], w1[r], direction)
        emulated_exchange(w1, w0, self.l1)
        for r in range(P):
            self.stages[r].unpack(w0[r], out[r])
        return out
