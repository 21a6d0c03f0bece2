# NS = 256 rows groups through the TMA kernel with tensor stores (r256) vs the plain rows kernel
for i in 1 2; do for v in base r256; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 16,17 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
python scripts/sweep.py --sizes 24 --layouts split --variants default --batch 8 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
done; done
cp abvar/r256/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -x -k "65536 or 131072 or 16 or 17" > gpurun_out/r256_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r256_pytest.log
