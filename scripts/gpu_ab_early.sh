# 2^14: pass-1 twiddle bases fetched before the stage wait vs after exchange-1 write
D=gpurun_out/ab_early; mkdir -p $D
for v in base early base early; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 14 --layouts split,interleaved --variants default >> $D/$v.jsonl 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "16384 or tma1" > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for f in base early; do echo == $f; python -c "
import json
for l in open('$D/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
