# checkpoint after the twiddle-base / TMA-store changes: full GPU suite, bench, K3 sweep
bash scripts/gpu_checkpoint.sh
python scripts/sweep.py --sizes 16,17,18,19,20,21 --layouts split,interleaved --variants default > gpurun_out/ckpt/sweep_k3.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ckpt/sweep_k3.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
