# asymmetric two-group splits for 2^18..2^21: sp1 = 10+8 / 11+8 / 11+9 / 12+9, sp2 = 8+10 / 10+9 / 12+8 / 11+10
for v in sp1 sp2; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x -k "262144 or 524288 or 1048576 or 2097152 or 18 or 19 or 20 or 21" > gpurun_out/sp_pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 gpurun_out/sp_pytest_$v.log
done
for i in 1 2; do for v in base sp1 sp2; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 18,19,20,21 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['ms'], d['frac'])"
done; done
