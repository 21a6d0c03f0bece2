# per-launch K3 group times after the tensor-store epilogues and twiddle prefetch (ncu launch list), 1 GiB batches
D=gpurun_out/r2al; mkdir -p $D
for n in 16 17 18 19 20 21 22 23 24; do for L in split interleaved; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $D/l_${n}_$L.csv python scripts/sweep.py --sizes $n --layouts $L --steps 1 --warmup 1 > /dev/null 2>&1
done; done
python - <<'PY'
import csv, glob, os, collections
U = {'ns': 1e-9, 'us': 1e-6, 'ms': 1e-3, 'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'second': 1.0,
     'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
for f in sorted(glob.glob('gpurun_out/r2al/l_*.csv'), key=lambda s: (int(s.split('_')[-2]), s)):
    rows = [r for r in csv.DictReader(l for l in open(f) if l.startswith('"'))]
    per = collections.OrderedDict()
    for r in rows:
        v = float(r['Metric Value'].replace(',', '')) * U.get(r['Metric Unit'], 1.0)
        per.setdefault((r['ID'], r['Kernel Name'][:70]), {})[r['Metric Name']] = v
    last = collections.OrderedDict()
    for (i, k), m in per.items():
        last[k] = m
    print(os.path.basename(f))
    for k, m in last.items():
        t = m.get('gpu__time_duration.sum', 0); by = m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
        print('   %-70s %9.1f us %7.3f GB %6.0f GB/s' % (k, t * 1e6, by / 1e9, by / t / 1e9 if t else 0))
PY
