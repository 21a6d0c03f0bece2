run() { timeout 300 python scripts/sweep.py --sizes $2 --layouts split,interleaved --steps 30 2>&1 | grep '"n"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$1', d['n'], d['layout'], d['frac'], d['ms'], d['kernel'])"
}
cp paper_2308_00497_b200/lib/libfftgen_b200.so /tmp/base.so
run BASE 10,11
for v in vA vB vC; do cp paper_2308_00497_b200/lib_$v/libfftgen_b200.so paper_2308_00497_b200/lib/; run $v 10,11; done
cp /tmp/base.so paper_2308_00497_b200/lib/libfftgen_b200.so
