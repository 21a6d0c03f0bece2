D=gpurun_out/ab_17; mkdir -p $D
for i in 1 2; do for v in base cur; do
if [ $v = base ]; then cp abvar/base/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so; else cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so; fi
python scripts/sweep.py --sizes 17,18,19 --layouts split --variants default 2>&1 | grep '"n"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n'], d['layout'][:5], d['ms'], d['frac'], d['kernel'])"
done; done
cp abvar/cur.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/l17.csv python scripts/sweep.py --sizes 17 --layouts split --steps 1 --warmup 1 > /dev/null 2>&1
grep fft_group $D/l17.csv | tail -2 | cut -d, -f5,15
cp abvar/base/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/l17b.csv python scripts/sweep.py --sizes 17 --layouts split --steps 1 --warmup 1 > /dev/null 2>&1
grep fft_group $D/l17b.csv | tail -2 | cut -d, -f5,15
