# per-launch times of 2^24 split: two-pass (tuning 16) vs the default three-pass, batch 8
D=gpurun_out/r2aj; mkdir -p $D
for v in default tuning=16; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $D/l_$v.csv python scripts/sweep.py --sizes 24 --layouts split --variants $v --batch 8 --steps 1 --warmup 1 > /dev/null 2>&1
done
ls $D
