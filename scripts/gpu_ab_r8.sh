# A/B: radix-8 three-pass plans as the default for 2^7..2^9 (abvar/r8), TMA and direct
mkdir -p gpurun_out/ab_r8
python scripts/sweep.py --sizes 7,8,9 --layouts split,interleaved --variants default,tuning=1,pass_radix=8 --steps 50 > gpurun_out/ab_r8/base.jsonl 2>&1
cp abvar/r8/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 7,8,9 --layouts split,interleaved --variants default,tuning=1 --steps 50 > gpurun_out/ab_r8/r8.jsonl 2>&1
for f in base r8; do echo == $f; python -c "
import json
for l in open('gpurun_out/ab_r8/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['ms'], d['frac'], d['kernel'])"; done
