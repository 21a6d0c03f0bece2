# K2r: new parity test + sanitizers over the small sizes
D=gpurun_out/r2ad; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "row_kernel" > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize.py > $D/$t.txt 2>&1
  echo "$t rc=$? $(tail -1 $D/$t.txt)"
done
