mkdir -p gpurun_out/r2o
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_matrix.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py -q > gpurun_out/r2o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2o/pytest.log
timeout 600 python scripts/sweep.py --sizes 6,7,8,9,10 --layouts split,interleaved --variants default,pass_radix=64 > gpurun_out/r2o/sweep.jsonl 2>&1
timeout 600 python scripts/sweep.py --sizes 7,8,9 --layouts split,interleaved --variants default --inverse > gpurun_out/r2o/sweep_inv.jsonl 2>&1
cat gpurun_out/r2o/sweep.jsonl gpurun_out/r2o/sweep_inv.jsonl | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['ms'], d['frac'], d['kernel'])"
