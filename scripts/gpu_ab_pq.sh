mkdir -p gpurun_out/ab_pq
python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default,tuning=20 > gpurun_out/ab_pq/base.jsonl 2>&1
cp abvar/pq/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default,tuning=20 > gpurun_out/ab_pq/pq.jsonl 2>&1
for f in base pq; do echo == $f; python -c "
import json
for l in open('gpurun_out/ab_pq/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
