# K2r final form: sweep 2^3..2^6 twice + the block-size parity tests
D=gpurun_out/r2ac; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_matrix.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_inputs.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for i in 1 2; do
python scripts/sweep.py --sizes 3,4,5,6,7 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
done
