timeout 600 python -m pytest tests/test_gpu_fourstep.py -x -q -k "phased" 2>&1 | tail -3
timeout 400 python scripts/sweep.py --sizes 15,16,18,20 --layouts interleaved,split --variants default,FFTGEN_PHASED=2+FFTGEN_DISABLE_CLUSTER=1+FFTGEN_PHASE_LAG=2+FFTGEN_PHASE_SLOT_MB=8,FFTGEN_PHASED=2+FFTGEN_DISABLE_CLUSTER=1+FFTGEN_PHASE_LAG=3+FFTGEN_PHASE_SLOT_MB=8,FFTGEN_PHASED=2+FFTGEN_DISABLE_CLUSTER=1+FFTGEN_PHASE_LAG=4+FFTGEN_PHASE_SLOT_MB=6,FFTGEN_PHASED=2+FFTGEN_DISABLE_CLUSTER=1+FFTGEN_PHASE_LAG=6+FFTGEN_PHASE_SLOT_MB=4 --steps 20 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
