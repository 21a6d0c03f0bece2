timeout 400 python scripts/sweep.py --sizes 15,16,17,18,20 --layouts split,interleaved --variants default,FFTGEN_PHASED=1+FFTGEN_DISABLE_CLUSTER=1,FFTGEN_PHASED=1+FFTGEN_DISABLE_CLUSTER=1+FFTGEN_PHASE_SLOT_MB=32 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
