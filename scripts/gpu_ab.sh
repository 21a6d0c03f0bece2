timeout 300 python scripts/sweep.py --sizes 16,18,20,24 --layouts split,interleaved --variants FFTGEN_GROUP_TMA=1+FFTGEN_PHASED=0 --batch 0 --steps 20 2>&1 | tail -10
cp paper_2308_00497_b200/lib_s1/libfftgen_b200.so paper_2308_00497_b200/lib/
timeout 300 python -m pytest tests/test_gpu_fourstep.py -q -x -k "group_tma" 2>&1 | tail -2
timeout 300 python scripts/sweep.py --sizes 16,18,20,24 --layouts split,interleaved --variants FFTGEN_GROUP_TMA=1+FFTGEN_PHASED=0 --steps 20 2>&1 | tail -10
