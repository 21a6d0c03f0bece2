# N = 4096 as three radix-16 passes (register twiddle bases) on the TMA kernel: one transform per CTA (p16a)
# or 64 KB double-buffered groups (p16b) vs the default 64 x 64 plan
D=gpurun_out/ab_p16; mkdir -p $D
for i in 1 2; do for v in base p16a p16b; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 12 --layouts split,interleaved --variants default --batch 65536 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
python scripts/sweep.py --sizes 12 --layouts split,interleaved --variants default --batch 4096 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
done; done
for v in p16a p16b; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "4096" > $D/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $D/pytest_$v.log
done
