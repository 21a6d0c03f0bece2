run() { timeout 300 python scripts/sweep.py --sizes 15,16,17,18,20 --layouts split,interleaved --variants default,FFTGEN_GROUP_TMA=0,FFTGEN_DISABLE_CLUSTER=1 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['kernel'])"
  timeout 300 python scripts/sweep.py --sizes 24 --batch 8 --layouts split,interleaved --variants default,FFTGEN_GROUP_TMA=0 --steps 10 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['kernel'])"
  timeout 300 python scripts/sweep.py --sizes 30 --batch 1 --layouts split,interleaved --variants default,FFTGEN_GROUP_TMA=0 --steps 4 --warmup 2 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
}
run T32
cp paper_2308_00497_b200/lib_t16/libfftgen_b200.so paper_2308_00497_b200/lib/
run T16
