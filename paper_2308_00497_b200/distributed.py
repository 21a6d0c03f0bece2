"""Multi-GPU partitioning of the FFT hot path, one process per GPU.

* BatchShardedFFT -- batched transforms (configs C2/C3) shard by contiguous
  batch ranges; every rank owns its own plan and twiddle tables and there is
  NO data-path collective (weak scaling).
* DistributedFFT  -- one very large transform (config C5, N = 2^30) block
  distributed over P ranks: the reference's Eq. 1 split
  DFT_N = (DFT_N1 (x) I) D^N (I (x) DFT_N2) Pi^N_N1 (formula.hpp:102-106) run
  as a distributed four-step with three all-to-all exchanges (NCCL over
  NVLink on GPUs; any torch.distributed backend works):

    rank r holds x[r M : (r+1) M], M = N/P, viewed as rows a of X[a][c] (N1 x N2)
    1. all-to-all: rank r gets columns c in [r N2/P, (r+1) N2/P) of every row
    2. N1-point FFTs down those columns            (local batched plan)
    3. twiddle D^N: F[c][k1] *= w_N^{c k1}          (fftgen_twiddle_multiply)
    4. all-to-all: rank r gets k1 in [r N1/P, (r+1) N1/P) for every c
    5. N2-point FFTs along c                        (local batched plan)
    6. all-to-all back to natural order: rank r ends with X^[r M : (r+1) M]

  Packing into per-peer contiguous chunks and the local transposes are
  strided tensor copies; the FFT passes are the sm_100a kernels.  The local
  FFT and the twiddle are injectable so the exchange logic is testable on
  CPU with the gloo backend (tests/test_distributed.py) against the oracle.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import FORWARD, PipelineConfig, compile_pipeline, twiddle_multiply


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


class DistributedFFT:
    """One N-point transform block-distributed over the process group."""

    def __init__(self, n: int, group=None, n1: Optional[int] = None, device: Optional[int] = None,
                 local_fft: Optional[Callable] = None, twiddle: Optional[Callable] = None):
        self.group = group
        self.rank, self.world = _rank_world(group)
        if n < 4 or n & (n - 1):
            raise ValueError(f"n must be a power of two >= 4, got {n}")
        log2 = n.bit_length() - 1
        self.n = n
        self.n1 = n1 or 1 << ((log2 + 1) // 2)
        self.n2 = n // self.n1
        P = self.world
        if self.n1 * self.n2 != n or self.n1 % P or self.n2 % P:
            raise ValueError(f"world size {P} must divide both factors {self.n1} x {self.n2}")
        self.m = n // P
        self._plans: dict = {}
        self.device = device
        self.local_fft = local_fft or self._gpu_fft
        self.twiddle = twiddle or (lambda blk, ro, co, nn, d: twiddle_multiply(blk, ro, co, nn, d))

    # ---- default GPU building blocks --------------------------------------
    def _gpu_fft(self, x: torch.Tensor, size: int, direction: int) -> torch.Tensor:
        """Batched contiguous complex64 FFTs of `size` along the last axis."""
        batch = x.shape[0]
        key = (size, batch)
        if key not in self._plans:
            dev = x.device.index if self.device is None else self.device
            self._plans[key] = compile_pipeline(PipelineConfig(n=size, batch=batch, layout="interleaved",
                                                               device=dev, algorithm="stockham"))
        out = torch.empty_like(x)
        self._plans[key].execute(x, out, direction=direction)
        return out

    def _a2a(self, send: torch.Tensor) -> torch.Tensor:
        recv = torch.empty_like(send)
        if self.world == 1:
            recv.copy_(send)
        else:
            dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), group=self.group)
        return recv

    # ---- the distributed four-step ----------------------------------------
    def execute(self, x_local: torch.Tensor, direction: int = FORWARD) -> torch.Tensor:
        """x_local: complex64 (M,) = x[rank*M : (rank+1)*M]; returns X^ of the same block."""
        P, r, N1, N2 = self.world, self.rank, self.n1, self.n2
        if x_local.numel() != self.m or x_local.dtype != torch.complex64:
            raise ValueError(f"expected complex64 block of {self.m} elements")
        if P == 1 and self.local_fft == self._gpu_fft:
            # nothing to exchange: the single-GPU K3 plan is the whole transform
            return self.local_fft(x_local.reshape(1, -1), self.n, direction).reshape(-1)
        X = x_local.reshape(N1 // P, N2)
        # 1. columns to their owners: chunk q = rows(r) x cols(q)
        R1 = self._a2a(X.reshape(N1 // P, P, N2 // P).transpose(0, 1).contiguous())
        del X
        Z = R1.reshape(N1, N2 // P).t().contiguous()          # (N2/P, N1): column c_loc contiguous
        del R1
        # 2. N1-point FFTs along a
        F = self.local_fft(Z, N1, direction)                   # F[c_loc][k1]
        del Z
        # 3. twiddle diagonal: c = r N2/P + c_loc, k1
        self.twiddle(F, r * (N2 // P), 0, self.n, direction)
        # 4. k1 ranges to their owners
        R2 = self._a2a(F.reshape(N2 // P, P, N1 // P).transpose(0, 1).contiguous())
        del F
        H = R2.reshape(N2, N1 // P).t().contiguous()          # (N1/P, N2): row k1_loc contiguous
        del R2
        # 5. N2-point FFTs along c
        O = self.local_fft(H, N2, direction)                   # O[k1_loc][k2]
        del H
        # 6. natural order: k = k1 + N1 k2, rank s owns k2 in [s N2/P, (s+1) N2/P)
        R3 = self._a2a(O.reshape(N1 // P, P, N2 // P).transpose(0, 1).contiguous())
        del O
        return R3.reshape(N1, N2 // P).t().contiguous().reshape(-1)
