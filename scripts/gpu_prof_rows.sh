# ncu --set full of the K3 row groups at 2^18 (NS=512) and 2^16 (NS=256), interleaved
D=gpurun_out/r1h; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fft_group_kernel -s 1 -c 1 -o $D/group_rows512_262144_il -f python scripts/sweep.py --sizes 18 --layouts interleaved --steps 1 --warmup 1 > /dev/null 2>&1
timeout 600 $NCU -k regex:fft_group_kernel -s 3 -c 1 -o $D/group_rows256_65536_il -f python scripts/sweep.py --sizes 16 --layouts interleaved --steps 1 --warmup 1 > /dev/null 2>&1
ls -la $D
