timeout 400 python scripts/sweep.py --sizes 15,16 --layouts split,interleaved --variants default,FFTGEN_CLUSTER_VARIANT=2,FFTGEN_CLUSTER_VARIANT=2+FFTGEN_CLUSTER_SIZE=4,FFTGEN_CLUSTER_VARIANT=2+FFTGEN_CLUSTER_SIZE=8,FFTGEN_CLUSTER_VARIANT=2+FFTGEN_CLUSTER_SIZE=16 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'][-40:], d['frac'], d['ms'], d['kernel'], d['bitwise_eq_first'])"
timeout 300 python scripts/sweep.py --sizes 14 --layouts split,interleaved --variants default,FFTGEN_CLUSTER14=1+FFTGEN_CLUSTER_VARIANT=2+FFTGEN_CLUSTER_SIZE=2,FFTGEN_CLUSTER14=1+FFTGEN_CLUSTER_VARIANT=2+FFTGEN_CLUSTER_SIZE=4 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'][-40:], d['frac'], d['ms'], d['kernel'], d['bitwise_eq_first'])"
