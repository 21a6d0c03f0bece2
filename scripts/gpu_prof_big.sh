# ncu: per-launch times and full captures of the NS = 2^12 group kernels (2-pass 2^24)
# vs the 3-pass NS = 2^8 groups, interleaved, batch 8
mkdir -p gpurun_out/r2c
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_2p24.csv python scripts/sweep.py --sizes 24 --layouts interleaved --variants tuning=16,tuning=8 --steps 2 --warmup 1 > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_group -s 2 -c 2 -o gpurun_out/r2c/group4096_2p24_il -f python scripts/sweep.py --sizes 24 --layouts interleaved --variants tuning=16 --steps 1 --warmup 1 > /dev/null 2>&1; echo "full rc=$?"
ls -la gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x -k "two_pass or plan_shape or three_group" > gpurun_out/r2c/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2c/pytest.log
