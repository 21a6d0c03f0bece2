timeout 600 python -m pytest tests/test_gpu_fourstep.py -x -q -k "phased or plan_shape" 2>&1 | tail -5
timeout 400 python scripts/sweep.py --sizes 16,18,20 --layouts split,interleaved --variants default,FFTGEN_PHASE_SLOT_MB=8,FFTGEN_PHASE_SLOT_MB=32,FFTGEN_PHASED=0 --steps 20 2>&1 | tail -40
