D=gpurun_out/r1d; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block_tma -s 2 -c 1 -o $D/block_tma_8192_split -f python scripts/sweep.py --sizes 13 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block_tma -s 2 -c 1 -o $D/block_tma_2048_split -f python scripts/sweep.py --sizes 11 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
ls $D
