# QFact also for NS = 512 / 1024 groups (q512) vs NS >= 2048 only (base)
cp abvar/q512/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x > gpurun_out/q512_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/q512_pytest.log
for i in 1 2; do for v in base q512; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 17,18,19,20,21 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'])"
done; done
