set -x
timeout 300 python scripts/sweep.py --sizes 14 --layouts split,interleaved --variants default,FFTGEN_CLUSTER14=1,FFTGEN_CLUSTER14=1+FFTGEN_CLUSTER_SIZE=2 --steps 20 2>&1 | tail -20
timeout 300 python scripts/sweep.py --sizes 15 --layouts split,interleaved --variants default,FFTGEN_CLUSTER_SIZE=4,FFTGEN_DISABLE_CLUSTER=1 --steps 20 2>&1 | tail -30
timeout 300 python scripts/sweep.py --sizes 16 --layouts split,interleaved --variants default,FFTGEN_CLUSTER_SIZE=8,FFTGEN_DISABLE_CLUSTER=1 --steps 20 2>&1 | tail -30
timeout 300 python scripts/sweep.py --sizes 17 --layouts split,interleaved --variants default,FFTGEN_DISABLE_CLUSTER=1 --steps 20 2>&1 | tail -30
python -c "
import paper_2308_00497_b200 as fg
for n in (1<<14, 1<<15, 1<<16, 1<<17):
    print(fg.compile_pipeline(fg.PipelineConfig(n=n, batch=64)).describe())
"
timeout 600 python -m pytest tests/test_gpu_fourstep.py -x -q -k "cluster or matches_oracle or plan_shape" 2>&1 | tail -15
