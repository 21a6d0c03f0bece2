# checkpoint + sweep refresh after the 2^14 epilogue and K3 twiddle prefetch
bash scripts/gpu_checkpoint.sh
bash scripts/gpu_sweep_r2.sh
