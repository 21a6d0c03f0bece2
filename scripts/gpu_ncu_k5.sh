mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_cluster -s 2 -c 1 -o gpurun_out/k5v2_32768_il -f \
  python scripts/sweep.py --sizes 15 --layouts interleaved --steps 1 --warmup 2 > gpurun_out/ncu_k5.log 2>&1
timeout 300 python scripts/sweep.py --sizes 14 --layouts interleaved --variants default,FFTGEN_CLUSTER14=1 --steps 20 --warmup 3 >> gpurun_out/ncu_k5.log 2>&1
tail -8 gpurun_out/ncu_k5.log
