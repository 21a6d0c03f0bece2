for spec in "16 interleaved 2048" "16 split 2048" "17 split 1024" "17 interleaved 1024"; do
set -- $spec
timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fft_group --csv \
  python scripts/sweep.py --sizes $1 --layouts $2 --batch $3 --steps 1 --warmup 1 2>/dev/null | grep fft_group | \
  python -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
out={}
for r in rows:
    try: out.setdefault((r[4].split('(')[0][-40:], r[-3]), []).append(r[-1])
    except Exception: pass
for k,v in out.items(): print('N=2^$1 $2', k, v[:2])
"
done
