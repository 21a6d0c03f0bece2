# ncu --set full of the small-N direct kernel, split vs interleaved (N = 64)
D=gpurun_out/r1k; mkdir -p $D
for L in split interleaved; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block -s 2 -c 1 -o $D/block_64_$L -f python scripts/sweep.py --sizes 6 --layouts $L --steps 1 --warmup 2 > /dev/null 2>&1
done
ls -la $D
