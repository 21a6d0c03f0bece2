mkdir -p gpurun_out/r2w
timeout 1500 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_distributed.py tests/test_gpu_twiddles.py -q > gpurun_out/r2w/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2w/pytest.log
( python scripts/sweep.py --sizes 15,16,17,18,19,20,21,22,23 --layouts split,interleaved 2>&1
  python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default,tuning=16 --batch 8 --steps 10 2>&1
  python scripts/sweep.py --sizes 24,26,28,30 --layouts split,interleaved --batch 1 --steps 5 --warmup 3 2>&1 ) > gpurun_out/r2w/sweep.jsonl
python -c "
import json
for l in open('gpurun_out/r2w/sweep.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['launches'], d['kernel'])"
