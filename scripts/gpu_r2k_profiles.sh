# round-2 ncu evidence: launch list of the default bench, full captures of the headline kernel,
# the NS=1024 group kernels after the stride search, the distributed stage kernels
D=gpurun_out/r2k; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 $NCU -k regex:fft_block_tma -s 3 -c 1 -o $D/block_tma_4096_split -f python bench.py --profile --steps 1 --warmup 4 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "headline rc=$?"
timeout 600 $NCU -k regex:fft_group -s 2 -c 2 -o $D/group1024_2p20_il -f python scripts/sweep.py --sizes 20 --layouts interleaved --steps 1 --warmup 1 > /dev/null 2>&1; echo "group rc=$?"
timeout 600 $NCU -k regex:dist_ -c 4 -o $D/dist_stages_2p28_p4 -f python scripts/dist_profile.py > /dev/null 2>&1; echo "dist rc=$?"
ls -la $D
