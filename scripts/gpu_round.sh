set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
cat gpurun_out/bench_default.json
for n in 16384 32768 65536 262144 1048576; do
  b=$((134217728 / n))
  timeout 300 python bench.py --n $n --batch $b --no-cpu-baseline --steps 50 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('N=$n', d['value'], d['roofline']['frac'], d['ms_per_step'])"
  FFTGEN_ENABLE_FLOW=1 timeout 300 python bench.py --n $n --batch $b --no-cpu-baseline --steps 50 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('FLOW N=$n', d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
