# ncu --set full of the opt-in K7 split-cluster kernel at 2^15
D=gpurun_out/r1i; mkdir -p $D
FFTGEN_SPLIT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_split -s 2 -c 1 -o $D/split_32768_il -f python scripts/sweep.py --sizes 15 --layouts interleaved --steps 1 --warmup 2 > /dev/null 2>&1
ls -la $D
