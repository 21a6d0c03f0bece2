# validation after QFact / twiddle prefetch / 2^14 epilogue: checkpoint, sanitizers, sweep
bash scripts/gpu_checkpoint.sh
D=gpurun_out/r2am_san; mkdir -p $D
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t python scripts/sanitize.py > $D/$t.txt 2>&1
  echo "$t rc=$? $(tail -1 $D/$t.txt)"
done
bash scripts/gpu_sweep_r2.sh
