# TwCache3 in the K2 kernels: block parity / matrix / edge tests + 2^7..2^13 sweep
D=gpurun_out/r2x; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_matrix.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest.log
timeout 600 python scripts/sweep.py --sizes 7,8,9,10,11,12,13 --layouts split,interleaved --variants default,pass_radix=16 > $D/sweep.jsonl 2>&1
python -c "
import json
for l in open('$D/sweep.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
