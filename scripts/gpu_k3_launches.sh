# per-launch times of the K3 group kernels (ncu launch list) for 2^17..2^20 and 2^24
mkdir -p gpurun_out/k3
for n in 17 18 20; do for L in split interleaved; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k3/l_${n}_$L.csv python scripts/sweep.py --sizes $n --layouts $L --steps 2 --warmup 1 > /dev/null 2>&1
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k3/l_24_split.csv python scripts/sweep.py --sizes 24 --layouts split --batch 8 --steps 2 --warmup 1 > /dev/null 2>&1
ls gpurun_out/k3
