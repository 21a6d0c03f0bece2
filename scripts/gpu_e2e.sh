mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'], d['e2e'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block -s 2 -c 1 -o gpurun_out/k2_16384_split -f \
  python scripts/sweep.py --sizes 14 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
ls gpurun_out
