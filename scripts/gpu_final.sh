# end-of-session validation: smoke, GPU tests, sanitizers (incl. opt-in paths),
# default bench, full sweep, launch list + ncu of the headline kernel
mkdir -p gpurun_out/final gpurun_out/san
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final/pytest_gpu.log
for t in memcheck racecheck synccheck; do
  SANITIZE_OPTIN=1 timeout 900 compute-sanitizer --tool $t python scripts/sanitize.py > gpurun_out/san/$t.txt 2>&1
  echo "$t rc=$? $(tail -1 gpurun_out/san/$t.txt)"
done
timeout 600 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo "bench rc=$?"
bash scripts/gpu_sweep_all.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block_tma -s 3 -c 1 -o gpurun_out/final/block_tma_4096_split -f python bench.py --profile --steps 1 --warmup 4 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_block -s 2 -c 1 -o gpurun_out/final/block_tma1_16384_il -f python scripts/sweep.py --sizes 14 --layouts interleaved --steps 1 --warmup 2 > /dev/null 2>&1
ls gpurun_out/final
