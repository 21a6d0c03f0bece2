# 2^14 kernel change: full GPU suite, sanitizers on the small cases, sweep
python -m pytest tests -x -q -m gpu 2>&1 | tail -2
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  SANITIZE_OPTIN=1 timeout 900 compute-sanitizer --tool $t python scripts/sanitize.py > gpurun_out/san/$t.txt 2>&1
  echo "$t rc=$? $(tail -1 gpurun_out/san/$t.txt)"
done
python scripts/sweep.py --sizes 12,13,14,15 2>&1 | grep '"n"' | cut -c1-140
