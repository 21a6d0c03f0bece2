D=gpurun_out/r2af; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block -s 2 -c 1 -o $D/block_2p14_split -f python scripts/sweep.py --sizes 14 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1; echo "14s rc=$?"
