timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -x -k "chunked" 2>&1 | tail -2
timeout 400 python scripts/sweep.py --sizes 15,16,17,18,20 --layouts split,interleaved --variants default,FFTGEN_DISABLE_CLUSTER=1+FFTGEN_L2_CHUNK_BYTES=16777216,FFTGEN_DISABLE_CLUSTER=1+FFTGEN_L2_CHUNK_BYTES=33554432,FFTGEN_DISABLE_CLUSTER=1+FFTGEN_L2_CHUNK_BYTES=50331648 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'][-30:], d['frac'], d['ms'], d['kernel'], d['bitwise_eq_first'])"
