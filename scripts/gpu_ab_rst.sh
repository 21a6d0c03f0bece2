# K3 rows groups (NS 2^9 / 2^10) through the TMA kernel with staged tensor stores (rst), or with
# register stores (rtma), vs the plain rows kernel (base); column groups unchanged
D=gpurun_out/ab_rst; mkdir -p $D
cp abvar/rst/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py -q -x -k "fourstep or rows or group" > $D/pytest_rst.log 2>&1; echo "pytest rst rc=$?"; tail -2 $D/pytest_rst.log
for i in 1 2; do for v in base rst rtma; do
cp abvar/$v/libfftgen_b200.so paper_2308_00497_b200/lib/libfftgen_b200.so
python scripts/sweep.py --sizes 16,17,18,19,20,21 --layouts split,interleaved --variants default >> $D/$v.jsonl 2>&1
done; done
for f in base rst rtma; do echo == $f; python -c "
import json
for l in open('$D/$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"; done
