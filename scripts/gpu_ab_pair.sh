# N = 64 by thread pairs (32-point halves + radix-2 combine through the row) vs one thread per transform
cp abvar/pair/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_matrix.py -q -x -k "row_kernel or block_sizes" > gpurun_out/pair_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pair_pytest.log
for i in 1 2; do for v in base pair; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 6 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'])"
done; done
