"""ncu target: the distributed four-step stages (butterfly / unpack, NCCL-chunk
and peer-pointer variants) at N = 2^28 with 4 ranks emulated on one GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_00497_b200.distributed import EmulatedDistributedFFT  # noqa: E402

n, world = 1 << 28, 4
m = n // world
blocks = [torch.complex(torch.rand(m, device="cuda"), torch.rand(m, device="cuda")) for _ in range(world)]
for t in ("nccl", "p2p"):
    EmulatedDistributedFFT(n, world, transport=t).execute(blocks)
torch.cuda.synchronize()
