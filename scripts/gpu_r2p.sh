mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_matrix.py -q -x -k "radix_hint" > gpurun_out/r2p/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2p/pytest.log
timeout 600 python scripts/sweep.py --sizes 10,11,12,13,14 --layouts split,interleaved --variants default,pass_radix=8,pass_radix=16 > gpurun_out/r2p/sweep.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2p/sweep.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['layout'][:5], d['variant'], d['ms'], d['frac'], d['kernel'])"
