# K3 TMA group kernel: pass-0 twiddles fetched before the stage wait (tp1: rows groups, tp2: all) vs base
for i in 1 2; do for v in base tp1 tp2; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 17,18,19,20,21 --layouts split,interleaved --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['batch'], d['ms'], d['frac'], d['kernel'])"
done; done
