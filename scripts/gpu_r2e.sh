# group exchange stride search (REG): parity + sweep 2^16..2^24 default and two-pass
mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_fuzz.py -q -x > gpurun_out/r2e/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2e/pytest.log
timeout 900 python scripts/sweep.py --sizes 16,17,18,19,20,21,22,23,24 --layouts split,interleaved --variants default,tuning=16 > gpurun_out/r2e/sweep.jsonl 2>&1
timeout 300 python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default,tuning=16 --batch 1 --steps 50 > gpurun_out/r2e/sweep_b1.jsonl 2>&1
cat gpurun_out/r2e/sweep.jsonl gpurun_out/r2e/sweep_b1.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['launches'], d['kernel'])"
