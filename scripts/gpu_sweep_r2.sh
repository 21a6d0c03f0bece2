mkdir -p gpurun_out
( timeout 600 python scripts/sweep.py --sizes 3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,18,19,20,21 --layouts split,interleaved --steps 30 2>&1 | grep '"n"'
  timeout 600 python scripts/sweep.py --sizes 7,8,9,10,12,14,16,18,20 --layouts split,interleaved --inverse --steps 30 2>&1 | grep '"n"' | sed 's/"variant": "default"/"variant": "inverse"/'
  timeout 300 python scripts/sweep.py --sizes 22,23,24 --layouts split,interleaved --steps 10 --warmup 3 2>&1 | grep '"n"'
  timeout 300 python scripts/sweep.py --sizes 21,22,23,24 --layouts split,interleaved --batch 8 --steps 10 --warmup 3 2>&1 | grep '"n"'
  timeout 300 python scripts/sweep.py --sizes 24,26,28,30 --layouts split,interleaved --batch 1 --steps 5 --warmup 3 2>&1 | grep '"n"' ) > gpurun_out/sweep_r2.jsonl
wc -l gpurun_out/sweep_r2.jsonl
