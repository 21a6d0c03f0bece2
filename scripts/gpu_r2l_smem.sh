# per-instruction shared-memory wavefronts of the K2 sizes the round-1 verdict flagged (2^6, 2^7, 2^13, 2^14)
D=gpurun_out/r2l; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
for spec in "13 split" "14 interleaved" "6 split" "6 interleaved" "7 split"; do
  set -- $spec
  timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_2p$1_$2 -f python scripts/sweep.py --sizes $1 --layouts $2 --steps 1 --warmup 2 > /dev/null 2>&1; echo "$spec rc=$?"
done
timeout 600 $NCU -k regex:dist_ -c 16 -o $D/dist_stages_2p28_p4 -f python scripts/dist_profile.py > /dev/null 2>&1; echo "dist rc=$?"
