# 2^19: NS=1024 rows group through the TMA kernel with tensor stores (cur) vs plain (base); 2^18/2^20 unchanged
D=gpurun_out/ab_r1024; mkdir -p $D
cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or rows or group" > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for i in 1 2; do for v in base cur; do
if [ $v = base ]; then cp abvar/base/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 18,19,20 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['ms'], d['frac'], d['kernel'])"
done; done
