# interleaved 2^10..2^12: default (2-pass TMA) vs pass_radix=16 (3-pass direct, cached twiddles), repeated
D=gpurun_out/ab_cap16; mkdir -p $D
for i in 1 2 3; do
python scripts/sweep.py --sizes 10,11,12 --layouts interleaved,split --variants default,pass_radix=16 >> $D/sweep.jsonl 2>&1
done
python scripts/sweep.py --sizes 10,11,12 --layouts interleaved --variants default,pass_radix=16 --bytes 16777216 >> $D/sweep.jsonl 2>&1
python scripts/sweep.py --sizes 10,11,12 --layouts interleaved --variants default,pass_radix=16 --bytes 134217728 >> $D/sweep.jsonl 2>&1
python -c "
import json
for l in open('$D/sweep.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:150]); continue
    print(d['n'], d['layout'][:5], d['variant'], d['batch'], d['ms'], d['frac'], d['kernel'])"
