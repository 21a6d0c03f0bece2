# A/B: plane-exchange kernel also for NS = 1024 groups (abvar/p10) vs NS >= 2048 only
mkdir -p gpurun_out/ab_p10
python scripts/sweep.py --sizes 18,19,20,21,25,26 --layouts split,interleaved > gpurun_out/ab_p10/base.jsonl 2>&1
cp abvar/p10/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 18,19,20,21,25,26 --layouts split,interleaved > gpurun_out/ab_p10/p10.jsonl 2>&1
for f in base p10; do echo == $f; python -c "
import json
for l in open('gpurun_out/ab_p10/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
