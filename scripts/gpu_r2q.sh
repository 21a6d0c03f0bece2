mkdir -p gpurun_out/r2q
timeout 600 python scripts/sweep.py --sizes 8,9,10,11,12,13 --layouts split,interleaved --variants default,tuning=1,pass_radix=64,pass_radix=16,pass_radix=32 > gpurun_out/r2q/sweep.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2q/sweep.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['ms'], d['frac'], d['kernel'], d['bitwise_eq_first'])"
timeout 900 python -m pytest tests/test_gpu_matrix.py -q -x -k "radix_hint or full_dft" > gpurun_out/r2q/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q/pytest.log
