run() { timeout 300 python scripts/sweep.py --sizes 8,9,10,11,12,13 --layouts split,interleaved --variants default,FFTGEN_DISABLE_TMA_STORE=1 --steps 30 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
}
run S2
cp paper_2308_00497_b200/lib_k1/libfftgen_b200.so paper_2308_00497_b200/lib/
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
run S1
