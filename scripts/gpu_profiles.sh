# round-1 evidence: ncu --set full of default kernels + launch list of the bench command
D=gpurun_out/r1e; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fft_block_tma -s 3 -c 1 -o $D/block_tma_4096_split -f python bench.py --profile --steps 1 --warmup 4 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 $NCU -k regex:fft_block_tma -s 2 -c 1 -o $D/block_tma_1024_split -f python scripts/sweep.py --sizes 10 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
timeout 600 $NCU -k regex:fft_block_tma -s 2 -c 1 -o $D/block_tma_2048_il -f python scripts/sweep.py --sizes 11 --layouts interleaved --steps 1 --warmup 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la $D
