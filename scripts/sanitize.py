"""Small runs of every kernel family, for compute-sanitizer (development tool).

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2308_00497_b200 as fg

    cases = [(8, 5), (16, 301), (32, 129), (64, 5), (256, 7), (512, 3), (1024, 9), (2048, 5), (4096, 7), (8192, 3), (16384, 150),  # K2
             (1 << 15, 3), (1 << 16, 2), (1 << 18, 1), (1 << 19, 1), (1 << 20, 1), (1 << 21, 1),
             (1 << 22, 1), (1 << 23, 1)]  # K5, K3 (+TMA groups, tensor-store epilogues, plane kernels)
    # non-default kernel selections: (PipelineConfig overrides, n, batch)
    optin = [(dict(tuning=fg.TUNE_NO_TMA), 1 << 14, 3), (dict(tuning=fg.TUNE_NO_TMA_STORE), 1 << 14, 150),
             (dict(cluster_size=16), 1 << 16, 3), (dict(tuning=fg.TUNE_GROUP_TMA_ALL, cluster_size=-1), 1 << 16, 2),
             (dict(pass_radix=16), 4096, 3), (dict(pass_radix=8), 2048, 3), (dict(pass_radix=16), 1 << 14, 2),
             (dict(tuning=16), 1 << 22, 1), (dict(tuning=16 | 4), 1 << 24, 1)]
    runs = [({}, n, b) for n, b in cases] + (optin if os.environ.get("SANITIZE_OPTIN") else [])
    for env, n, batch in runs:
        for layout in ("interleaved", "split"):
            x = torch.rand(batch, n, 2, device="cuda") * 2 - 1
            plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch, **env))
            if layout == "interleaved":
                y = torch.empty_like(x)
                plan.execute(x, y)
                plan.execute(y, y, direction=fg.INVERSE)
            else:
                re, im = x[..., 0].contiguous(), x[..., 1].contiguous()
                ore, oim = torch.empty_like(re), torch.empty_like(im)
                plan.execute(re, ore, im, oim)
            torch.cuda.synchronize()
            print(env, n, batch, layout, plan.describe().splitlines()[2][:60], flush=True)
            plan.close()
    # device input generator and the distributed stages (NCCL-chunk and peer variants), 4 emulated ranks
    fg.seeded_input(4096, 3, "split")
    fg.seeded_input(1000, 2, "interleaved", dist=1003)
    from paper_2308_00497_b200.distributed import EmulatedDistributedFFT
    n, world = 1 << 16, 4
    blocks = [torch.complex(torch.rand(n // world, device="cuda"), torch.rand(n // world, device="cuda"))
              for _ in range(world)]
    for t in ("nccl", "p2p"):
        EmulatedDistributedFFT(n, world, transport=t).execute(blocks)
    torch.cuda.synchronize()
    print("seeded_input + distributed stages ok", flush=True)


if __name__ == "__main__":
    main()
