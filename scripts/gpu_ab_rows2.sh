# K2r: one tile per CTA (rows128) vs grid capped at 4 / 16 CTAs per SM with a tile loop
D=gpurun_out/ab_rows2; mkdir -p $D
for v in rows128 rc4 rc16; do
if [ $v = rows128 ]; then cp abvar/rows128.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "small or batch or 64 or 32" > $D/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $D/pytest_$v.log
python scripts/sweep.py --sizes 3,4,5,6 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
done
