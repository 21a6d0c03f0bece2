# twiddle prefetch per the measured rule (cur) vs base; parity of the group kernels
cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py tests/test_gpu_edge.py -q -x -k "fourstep or rows or group or epilog or unaligned or padded" > gpurun_out/tp_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/tp_pytest.log
for i in 1 2; do for v in base cur; do
if [ $v = base ]; then cp abvar/base/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 17,18,19,20,21 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'])"
done; done
