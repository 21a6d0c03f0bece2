# refresh: full sweep + ncu launch list of the default bench + headline capture summary
bash scripts/gpu_sweep_r2.sh
D=gpurun_out/r2ag; mkdir -p $D
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block_tma -s 3 -c 1 -o $D/block_tma_4096_split -f python bench.py --profile --steps 1 --warmup 4 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "headline rc=$?"
python profiles/summarize.py $D r2ag > $D/summarize.log 2>&1; echo "summarize rc=$?"
mkdir -p $D/txt && cp profiles/r2ag_* profiles/ncu_summary.json $D/txt/ 2>/dev/null; rm -f $D/*.ncu-rep; ls $D/txt
