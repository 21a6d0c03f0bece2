# round 2: new tests (inputs, distributed), default bench, reference arm, distributed bench at world 1
mkdir -p gpurun_out/r2a
timeout 900 python -m pytest tests/test_gpu_inputs.py tests/test_gpu_distributed.py -q -x > gpurun_out/r2a/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2a/pytest.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2a/ref.json 2> gpurun_out/r2a/ref.err; echo "ref rc=$?"
for l2 in 24 28 30; do
timeout 600 python bench.py --workload distributed --n $((1<<l2)) --steps 10 --warmup 3 > gpurun_out/r2a/dist_$l2.json 2> gpurun_out/r2a/dist_$l2.err; echo "dist $l2 rc=$?"
done
cat gpurun_out/r2a/*.json | cut -c1-600
