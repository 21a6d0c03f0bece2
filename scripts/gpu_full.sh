mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
cat gpurun_out/bench_default.json
timeout 300 python bench.py --layout interleaved --no-cpu-baseline --e2e-steps 1 | cut -c1-400
timeout 300 python bench.py --direction inverse --no-cpu-baseline --e2e-steps 1 | cut -c1-400
