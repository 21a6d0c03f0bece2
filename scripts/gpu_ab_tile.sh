# A/B: NS = 2^11 / 2^12 group tiles of 128 KB (default) vs 64 KB (abvar/tile64), two-pass plans
mkdir -p gpurun_out/ab_tile
python scripts/sweep.py --sizes 22,23,24 --layouts split,interleaved --variants tuning=16,tuning=17,tuning=20 > gpurun_out/ab_tile/t128.jsonl 2>&1
cp abvar/tile64/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 22,23,24 --layouts split,interleaved --variants tuning=16,tuning=17,tuning=20 > gpurun_out/ab_tile/t64.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -x -k two_pass > gpurun_out/ab_tile/pytest64.log 2>&1; echo "pytest64 rc=$?"
for f in t128 t64; do echo == $f; python -c "
import sys,json
for l in open('gpurun_out/ab_tile/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
