# K2r row kernel (N = 8..64, one transform per thread) with 64/128/256-thread CTAs vs the direct kernel (tuning=1)
D=gpurun_out/ab_rows; mkdir -p $D
cp abvar/rows128.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_matrix.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest.log
for v in rows128 r64 r256; do
if [ $v = rows128 ]; then cp abvar/rows128.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 3,4,5,6 --layouts split,interleaved --variants default,tuning=1 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
done
