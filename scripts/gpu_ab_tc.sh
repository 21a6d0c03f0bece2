# 2^13 K2 TMA with passes 1-2 twiddle bases cached in registers (TwCache3) vs table loads
D=gpurun_out/ab_tc; mkdir -p $D
for v in base tc; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 13 --layouts split,interleaved --variants default > $D/$v.jsonl 2>&1
python scripts/sweep.py --sizes 13 --layouts split,interleaved --variants default >> $D/$v.jsonl 2>&1
done
cp abvar/tc/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 600 python -m pytest tests/test_gpu_matrix.py -q -x -k "block_sizes and 13" > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for f in base tc; do echo == $f; python -c "
import json
for l in open('$D/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
