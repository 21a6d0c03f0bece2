FFTGEN_PHASED=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_stream -s 2 -c 1 -o gpurun_out/k6b_65536_il -f python scripts/sweep.py --sizes 16 --layouts interleaved --steps 1 --warmup 2 > /dev/null 2>&1
ls gpurun_out | grep k6b
