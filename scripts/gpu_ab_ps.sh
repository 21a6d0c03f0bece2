# plane kernel (NS 2^11/2^12): results by TMA tensor stores staged through the plane, rows (ps1) / all (ps2)
D=gpurun_out/ab_ps; mkdir -p $D
for v in ps1 ps2; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or rows or group" > $D/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -2 $D/pytest_$v.log
done
for i in 1 2; do for v in base ps1 ps2; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default --batch 1 --steps 50 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
done; done
