timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
timeout 400 python scripts/sweep.py --sizes 8,9,10,11,12,13 --layouts split,interleaved --steps 30 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['frac'], d['ms'], d['kernel'])"
