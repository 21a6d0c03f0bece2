# 2^14: last pass stored butterfly by butterfly (sj: butterfly 0's bulk stores overlap butterfly 1's compute) vs halves
for i in 1 2; do for v in base sj; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 14 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
done; done
cp abvar/sj/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_matrix.py -q -x -k "16384 or tma1 or in_place or 14" > gpurun_out/sj_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/sj_pytest.log
