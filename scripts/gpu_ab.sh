run() { timeout 300 python scripts/sweep.py --sizes 17,18,19,20 --layouts split,interleaved --variants default,FFTGEN_GROUP_TMA=0 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
  timeout 300 python scripts/sweep.py --sizes 25,28 --batch 1 --layouts split,interleaved --steps 5 --warmup 2 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
}
cp paper_2308_00497_b200/lib/libfftgen_b200.so /tmp/base.so
run BASE
cp paper_2308_00497_b200/lib_g3/libfftgen_b200.so paper_2308_00497_b200/lib/
timeout 600 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_fuzz.py -q -x -k "not phased" 2>&1 | tail -2
run G3
cp /tmp/base.so paper_2308_00497_b200/lib/libfftgen_b200.so
