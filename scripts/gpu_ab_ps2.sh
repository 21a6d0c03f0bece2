# plane-kernel tensor stores per the measured rule (cur) vs base; split two-pass 2^23/2^24 (tuning 16) with them
D=gpurun_out/ab_ps2; mkdir -p $D
cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or rows or group" > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for v in base cur; do
if [ $v = base ]; then cp abvar/base/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default,tuning=16 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default,tuning=16 --batch 1 --steps 50 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
done
