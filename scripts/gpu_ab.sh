run() { timeout 300 python scripts/sweep.py --sizes 12,11,13,10 --layouts split,interleaved --steps 30 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['variant'], d['frac'], d['ms'], d['kernel'])"
  python -c "
import paper_2308_00497_b200 as fg
print('$1', fg.compile_pipeline(fg.PipelineConfig(n=4096, layout='split', batch=65536)).describe().splitlines()[2])"
}
run CARVE
cp paper_2308_00497_b200/lib_m7/libfftgen_b200.so paper_2308_00497_b200/lib/
run CARVE_M7
