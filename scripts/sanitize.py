"""Small runs of every kernel family, for compute-sanitizer (development tool).

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2308_00497_b200 as fg

    cases = [(64, 5), (1024, 9), (2048, 5), (4096, 7), (8192, 3), (16384, 150),  # K2 direct / TMA
             (1 << 15, 3), (1 << 16, 2), (1 << 18, 1), (1 << 21, 1)]          # K5, K3 (+TMA groups)
    # opt-in paths: (env, n, batch)
    optin = [({"FFTGEN_PHASED": "1", "FFTGEN_PHASE_SLOT_MB": "1"}, 1 << 16, 5),
             ({"FFTGEN_PHASED": "2", "FFTGEN_PHASE_SLOT_MB": "1"}, 1 << 16, 5),
             ({"FFTGEN_CLUSTER14": "1"}, 1 << 14, 3), ({"FFTGEN_TMA1": "0"}, 1 << 14, 3),
             ({"FFTGEN_TMA1_EX1": "0", "FFTGEN_DISABLE_TMA_STORE": "0"}, 1 << 14, 150),
             ({"FFTGEN_SPLIT": "1"}, 1 << 15, 5), ({"FFTGEN_SPLIT": "1"}, 1 << 16, 3),
             ({"FFTGEN_GROUP_TMA": "1"}, 1 << 16, 2), ({"FFTGEN_L2_CHUNK_BYTES": "1048576",
                                                        "FFTGEN_DISABLE_CLUSTER": "1"}, 1 << 15, 9)]
    runs = [({}, n, b) for n, b in cases] + (optin if os.environ.get("SANITIZE_OPTIN") else [])
    for env, n, batch in runs:
        saved = dict(os.environ)
        os.environ.update(env)
        for layout in ("interleaved", "split"):
            x = torch.rand(batch, n, 2, device="cuda") * 2 - 1
            plan = fg.compile_pipeline(fg.PipelineConfig(n=n, layout=layout, batch=batch))
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
        os.environ.clear()
        os.environ.update(saved)


if __name__ == "__main__":
    main()
