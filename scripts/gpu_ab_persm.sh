# N = 4096 persistent TMA grid: 5 / 6 CTAs per SM (occupancy limit 6) vs the default 4
for i in 1 2; do for v in base ps5 ps6; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 12 --layouts split,interleaved --variants default --batch 65536 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
python -c "
import paper_2308_00497_b200 as fg
p=fg.compile_pipeline(fg.PipelineConfig(n=4096,batch=65536,layout='split')); print('$v', p.describe().splitlines()[2][:60])"
done; done
