# K3 group TMA kernel: staged TMA tensor stores (st) and rows groups through it (str) vs register STGs
D=gpurun_out/ab_st; mkdir -p $D
for v in st str; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or rows or group" > $D/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -2 $D/pytest_$v.log
done
for v in base st str; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 16,17,18,19,20,21 --layouts split,interleaved --variants default > $D/$v.jsonl 2>&1
done
for f in base st str; do echo == $f; python -c "
import json
for l in open('$D/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
