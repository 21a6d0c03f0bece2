timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_edge.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 400 python scripts/sweep.py --sizes 15 --layouts split,interleaved --variants default,FFTGEN_DISABLE_CLUSTER=1 --steps 20 2>&1 | grep '"n"'
timeout 400 python scripts/sweep.py --sizes 16,17,18,19,20 --layouts split,interleaved --steps 20 2>&1 | grep '"n"'
timeout 300 python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --batch 8 --steps 10 --warmup 2 2>&1 | grep '"n"'
timeout 300 python scripts/sweep.py --sizes 24 --layouts split,interleaved --batch 1 --steps 10 --warmup 2 2>&1 | grep '"n"'
timeout 300 python scripts/sweep.py --sizes 26,28,30 --layouts split,interleaved --batch 1 --steps 4 --warmup 2 2>&1 | grep '"n"'
