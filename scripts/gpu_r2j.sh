mkdir -p gpurun_out/r2j
for t in nccl p2p; do
timeout 600 python bench.py --workload distributed --transport $t --n $((1<<28)) --steps 10 --warmup 3 > gpurun_out/r2j/dist_$t.json 2> gpurun_out/r2j/dist_$t.err; echo "dist $t rc=$?"; tail -3 gpurun_out/r2j/dist_$t.err
done
python -c "
import json
for t in ('nccl','p2p'):
    d=json.loads(open(f'gpurun_out/r2j/dist_{t}.json').read().strip().splitlines()[-1]); print(t, d['ms_per_step'], d['stages_ms'], d['e2e']['value'])"
