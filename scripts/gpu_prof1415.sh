# ncu --set full of the 2^14 single-stage and 2^15 cluster kernels
D=gpurun_out/r1g; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_tma1_16384_interleaved -f python scripts/sweep.py --sizes 14 --layouts interleaved --steps 1 --warmup 2 > /dev/null 2>&1
timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_tma1_16384_split -f python scripts/sweep.py --sizes 14 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
timeout 600 $NCU -k regex:fft_cluster -s 2 -c 1 -o $D/cluster_32768_split -f python scripts/sweep.py --sizes 15 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
ls -la $D
