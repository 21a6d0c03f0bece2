# A/B: NS = 2^11 / 2^12 groups as 64-point two-pass (default) vs three 16-point passes on 1024 threads (abvar/big3)
mkdir -p gpurun_out/ab_big3
python scripts/sweep.py --sizes 22,23,24 --layouts split,interleaved --variants default,tuning=16,tuning=20 > gpurun_out/ab_big3/base.jsonl 2>&1
cp abvar/big3/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 22,23,24 --layouts split,interleaved --variants tuning=16,tuning=17,tuning=20 > gpurun_out/ab_big3/big3.jsonl 2>&1
python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default,tuning=16,tuning=20 --batch 1 --steps 50 > gpurun_out/ab_big3/big3_b1.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -x -k two_pass > gpurun_out/ab_big3/pytest.log 2>&1; echo "pytest big3 rc=$?"
for f in base big3 big3_b1; do echo == $f; python -c "
import json
for l in open('gpurun_out/ab_big3/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
