D=gpurun_out/r2ai; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block_tma -s 3 -c 1 -o $D/block_tma_4096_split -f python bench.py --profile --steps 1 --warmup 4 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "headline rc=$?"
