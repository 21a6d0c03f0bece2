# exchange microbenchmark (smem vs __shfl_xor_sync 32x32 warp transpose) + full sweep refresh
D=gpurun_out/r2z; mkdir -p $D
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $D/exchange_microbench tools/exchange_microbench.cu && \
  for i in 1 2; do $D/exchange_microbench; done > $D/exchange_microbench.jsonl 2>&1; cat $D/exchange_microbench.jsonl
bash scripts/gpu_sweep_r2.sh
