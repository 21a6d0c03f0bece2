# NS >= 2^11 groups: pass-0 Q twiddles as products of two loaded bases (qpq) vs one load per element
cp abvar/qpq/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or group or rows" > gpurun_out/qpq_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/qpq_pytest.log
for i in 1; do for v in base qpq; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'])"
python scripts/sweep.py --sizes 24 --layouts interleaved --variants default --batch 1 --steps 50 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'])"
done; done
