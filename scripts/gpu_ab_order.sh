# K3 group order: larger group first for 2^19 split / 2^21 interleaved (cur) vs base; 2^23 split as 12+11 (s23)
cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or rows or group" > gpurun_out/ord_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ord_pytest.log
for i in 1 2; do for v in base cur s23; do
if [ $v = cur ]; then cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 19,21,23 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['ms'], d['frac'])"
done; done
