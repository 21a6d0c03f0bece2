# two-group splits with small rows groups: sp3 = 9+7 / 10+7 / 11+7 / 12+7 (2^16..2^19), sp4 = 8+8 / 9+8 / 10+8 / 12+7
for v in sp3 sp4; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x -k "65536 or 131072 or 262144 or 524288 or 16 or 17 or 18 or 19" > gpurun_out/sp_pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 gpurun_out/sp_pytest_$v.log
done
for i in 1 2; do for v in base sp3 sp4; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 16,17,18,19 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['ms'], d['frac'])"
done; done
