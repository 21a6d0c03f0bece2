# sweep twice (run-to-run spread on one box)
bash scripts/gpu_sweep_r2.sh; cp gpurun_out/sweep_r2.jsonl gpurun_out/sweep_r2_a.jsonl
bash scripts/gpu_sweep_r2.sh; cp gpurun_out/sweep_r2.jsonl gpurun_out/sweep_r2_b.jsonl
