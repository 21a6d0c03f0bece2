mkdir -p gpurun_out/r2s
timeout 600 python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default,tuning=16,tuning=20,tuning=4 > gpurun_out/r2s/sweep.jsonl 2>&1
timeout 300 python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default,tuning=16,tuning=20 --batch 1 --steps 50 > gpurun_out/r2s/sweep_b1.jsonl 2>&1
cat gpurun_out/r2s/sweep.jsonl gpurun_out/r2s/sweep_b1.jsonl | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'], d['bitwise_eq_first'])"
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "two_pass or fourstep" > gpurun_out/r2s/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2s/pytest.log
