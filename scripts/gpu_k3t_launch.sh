for v in 1 0; do
for spec in "16 interleaved 2048" "16 split 2048" "18 split 512" "18 interleaved 512" "20 split 128" "20 interleaved 128" "24 split 8" "24 interleaved 8" "30 split 1"; do
set -- $spec
FFTGEN_DISABLE_CLUSTER=1 FFTGEN_GROUP_TMA=$v timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fft_group --csv \
  python scripts/sweep.py --sizes $1 --layouts $2 --batch $3 --steps 1 --warmup 1 2>/dev/null | grep fft_group | \
  python -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
ks={}
for r in rows:
    name=r[4] if len(r)>4 else ''
    try: ks.setdefault(name.split('(')[0][:60]+'|'+name.split('<')[1].split('>')[0], []).append(float(r[-1]))
    except Exception: pass
print('TMA=$v N=2^$1 $2', {k: round(min(v),1) for k,v in ks.items()})
"
done; done
