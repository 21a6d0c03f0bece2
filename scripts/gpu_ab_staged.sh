# direct radix-8 kernel with row-staged input (s1), + staged output (s2), up to 2^9 (s3) vs base
cp abvar/s3/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_matrix.py -q -x -k "128 or 256 or 512 or block_sizes or hint" > gpurun_out/st_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/st_pytest.log
for i in 1 2; do for v in base s1 s2 s3; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 7,8,9 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'])"
done; done
