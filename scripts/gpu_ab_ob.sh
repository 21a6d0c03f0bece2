# N = 4096: results staged in their own buffer, next load issued right after the exchange (ob, 3 CTAs/SM)
# vs the single-stage slot (base, 4 CTAs/SM); tuning=2 = register stores
cp abvar/ob/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "4096" > gpurun_out/ob_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ob_pytest.log
python -c "
import paper_2308_00497_b200 as fg
print(fg.compile_pipeline(fg.PipelineConfig(n=4096,batch=65536,layout='split')).describe().splitlines()[2][:90])"
for i in 1 2; do for v in base ob; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 12 --layouts split,interleaved --variants default,tuning=2 --batch 65536 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'])"
done; done
