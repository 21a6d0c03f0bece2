# checkpoint: smoke, full GPU suite, default bench, reference arm, distributed bench
D=gpurun_out/ckpt; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $D/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $D/ref.json 2> $D/ref.err; echo "ref rc=$?"
python -c "
import json
d=json.loads(open('$D/bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e'].get('vs_cpu'), d['clocks'])
r=json.loads(open('$D/ref.json').read().strip().splitlines()[-1]); print('ref', r['value'], r['ms_per_step'], r['config']['sample_transforms'])"
