# K5 (2^15) sub-FFTs with register pass-1 twiddle bases (k5pq) vs table loads (base)
for i in 1 2; do for v in base k5pq; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 15 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
done; done
cp abvar/k5pq/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_edge.py -q -x -k "32768 or cluster or 15" > gpurun_out/k5pq_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/k5pq_pytest.log
