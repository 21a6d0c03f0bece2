mkdir -p gpurun_out/r2n
timeout 900 python -m pytest tests/test_gpu_matrix.py -q -x -k "radix_hint" > gpurun_out/r2n/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2n/pytest.log
timeout 600 python scripts/sweep.py --sizes 7,8,9,10,11,12 --layouts split,interleaved --variants default,pass_radix=8,pass_radix=16,pass_radix=32 > gpurun_out/r2n/sweep.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2n/sweep.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['ms'], d['frac'], d['kernel'], d['bitwise_eq_first'])"
