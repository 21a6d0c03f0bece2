python scripts/pcie_probe.py
timeout 300 python scripts/sweep.py --sizes 18,19,20 --layouts split,interleaved --steps 20 2>&1 | tail -30
timeout 300 python scripts/sweep.py --sizes 28,30 --layouts split --variants default,FFTGEN_GROUP_MAX_LOG2=10 --batch 1 --steps 5 --warmup 2 2>&1 | tail -30
timeout 300 python scripts/sweep.py --sizes 24 --layouts split,interleaved --batch 8 --steps 10 --warmup 2 2>&1 | tail -30
