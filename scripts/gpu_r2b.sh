# 2-pass four-step for 2^21..2^24 (NS = 2^11 / 2^12 groups): parity + A/B sweep
mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x > gpurun_out/r2b/pytest_fourstep.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2b/pytest_fourstep.log
timeout 600 python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --variants default,tuning=8,tuning=1,tuning=4 --bytes 1073741824 > gpurun_out/r2b/sweep_1g.jsonl 2>&1
timeout 600 python scripts/sweep.py --sizes 24 --layouts split,interleaved --variants default,tuning=8,tuning=1,tuning=4 --batch 1 --steps 50 > gpurun_out/r2b/sweep_b1.jsonl 2>&1
cat gpurun_out/r2b/sweep_1g.jsonl gpurun_out/r2b/sweep_b1.jsonl | cut -c1-200
