# ncu --set full of the 2^14 kernels (direct and single-stage TMA) on one GPU
D=gpurun_out/r1f; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
for L in split interleaved; do
  FFTGEN_TMA1=1 timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_tma1_16384_$L -f python scripts/sweep.py --sizes 14 --layouts $L --steps 1 --warmup 2 > /dev/null 2>&1
done
timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_16384_split -f python scripts/sweep.py --sizes 14 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1
ls -la $D
