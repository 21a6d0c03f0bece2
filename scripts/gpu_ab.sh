run() { timeout 300 python scripts/sweep.py --sizes 14 --layouts split,interleaved --steps 30 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
}
run BASE
cp paper_2308_00497_b200/lib_a14/libfftgen_b200.so paper_2308_00497_b200/lib/
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
run ALT
