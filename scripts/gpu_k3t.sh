timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_edge.py -x -q 2>&1 | tail -5
timeout 400 python scripts/sweep.py --sizes 15,16,17,18,19,20 --layouts split,interleaved --steps 20 2>&1 | tail -30
timeout 300 python scripts/sweep.py --sizes 21,22,24 --layouts split,interleaved --batch 8 --steps 10 --warmup 2 2>&1 | tail -30
timeout 300 python scripts/sweep.py --sizes 30 --layouts split,interleaved --batch 1 --steps 5 --warmup 2 2>&1 | tail -30
