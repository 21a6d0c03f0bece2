# three / four-group splits at batch 1: current rules (cur) + candidates for 2^25 / 2^29 (t1: 8+8+9 / 8+10+11, t2: 7+8+10 / 8+9+12)
cp paper_2308_00497_b200/lib/libfftgen_b200.so abvar/cur.so
for v in base cur t1 t2; do
if [ $v = cur ]; then cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 25,26,27,28,29,30 --layouts split,interleaved --variants default --batch 1 --steps 5 --warmup 3 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['ms'], d['frac'], d['launches'])"
done
cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x > gpurun_out/s3_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3_pytest.log
