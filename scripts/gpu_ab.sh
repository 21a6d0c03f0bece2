timeout 300 python scripts/sweep.py --sizes 17,19 --layouts split,interleaved --variants default,FFTGEN_LARGE_FIRST=1 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
timeout 300 python scripts/sweep.py --sizes 21,22,23,25 --batch 8 --layouts split,interleaved --variants default,FFTGEN_LARGE_FIRST=1 --steps 10 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
timeout 300 python -m pytest tests/test_gpu_fourstep.py -q -x -k "matches_oracle or three_group" 2>&1 | tail -2
FFTGEN_LARGE_FIRST=1 timeout 300 python -m pytest tests/test_gpu_fourstep.py -q -x -k "matches_oracle or three_group" 2>&1 | tail -2
