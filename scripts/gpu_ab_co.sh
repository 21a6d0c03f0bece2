# N = 4096 TMA kernel with a larger shared-memory carveout (more resident CTAs): 100 % / 80 % vs default
for i in 1 2; do for v in base co100 co80; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 12 --layouts split,interleaved --variants default --batch 65536 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'], d.get('describe','')[:0])"
python -c "
import paper_2308_00497_b200 as fg
p=fg.compile_pipeline(fg.PipelineConfig(n=4096,batch=65536,layout='split')); print('$v', p.describe().splitlines()[2][:80])"
done; done
