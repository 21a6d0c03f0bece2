# compute-sanitizer after the tensor-store epilogues (K2 twiddle bases, K3 TMA stores, plane stores)
D=gpurun_out/r2ab_san; mkdir -p $D
for t in memcheck racecheck synccheck; do
  SANITIZE_OPTIN=1 timeout 1200 compute-sanitizer --tool $t python scripts/sanitize.py > $D/$t.txt 2>&1
  echo "$t rc=$? $(tail -1 $D/$t.txt)"
done
timeout 1200 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_matrix.py tests/test_gpu_parity.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
