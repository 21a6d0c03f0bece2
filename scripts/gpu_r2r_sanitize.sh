# compute-sanitizer over every kernel family incl. the round-2 kernels
D=gpurun_out/r2r_san; mkdir -p $D
for t in memcheck racecheck synccheck; do
  SANITIZE_OPTIN=1 timeout 1200 compute-sanitizer --tool $t python scripts/sanitize.py > $D/$t.txt 2>&1
  echo "$t rc=$? $(tail -1 $D/$t.txt)"
done
