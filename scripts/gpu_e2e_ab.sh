# e2e (fftgen_execute_host) host-pipeline chunking A/B on the C2 bench
for v in "FFTGEN_HOST_CHUNK_MB=128 FFTGEN_HOST_RAMP=4" "FFTGEN_HOST_CHUNK_MB=256" "FFTGEN_HOST_CHUNK_MB=256 FFTGEN_HOST_RAMP=5" "FFTGEN_HOST_CHUNK_MB=512 FFTGEN_HOST_RAMP=6" "FFTGEN_HOST_CHUNK_MB=256 FFTGEN_HOST_RAMP=3" "" ; do
  env $v timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v'.ljust(45), round(e['value'],1), round(e['ms_per_step'],2), e['roofline']['peak'], round(e['roofline']['frac'],3))"
done
