timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_phased -s 2 -c 1 -o gpurun_out/k6_65536_split -f python scripts/sweep.py --sizes 16 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
ls gpurun_out
