D=gpurun_out/r2t; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:fft_group_plane -s 2 -c 2 -o $D/plane4096_2p24_il -f python scripts/sweep.py --sizes 24 --layouts interleaved --variants tuning=20 --steps 1 --warmup 1 > /dev/null 2>&1; echo "4096 rc=$?"
timeout 900 $NCU -k regex:fft_group_plane -s 2 -c 2 -o $D/plane2048_2p22_il -f python scripts/sweep.py --sizes 22 --layouts interleaved --steps 1 --warmup 1 > /dev/null 2>&1; echo "2048 rc=$?"
