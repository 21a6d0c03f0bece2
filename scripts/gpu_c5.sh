timeout 300 python scripts/sweep.py --sizes 29,30 --layouts split,interleaved --batch 1 --variants default,FFTGEN_GROUP_MAX_LOG2=10,FFTGEN_GROUP_MAX_LOG2=10+FFTGEN_GROUP_TMA=1 --steps 4 --warmup 2 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['launches'], d['kernel'])"
