# ncu full captures after the round-2 K2 changes: 2^13 split (TwCache3), 2^14 split/interleaved (factored bases),
# 2^5 split (row kernel), 2^18 split rows group (TMA tensor stores), 2^24 interleaved plane rows (tensor stores)
D=gpurun_out/r2ae; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_2p13_split -f python scripts/sweep.py --sizes 13 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1; echo "13 rc=$?"
timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_2p14_split -f python scripts/sweep.py --sizes 14 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1; echo "14s rc=$?"
timeout 600 $NCU -k regex:fft_block -s 2 -c 1 -o $D/block_2p14_interleaved -f python scripts/sweep.py --sizes 14 --layouts interleaved --steps 1 --warmup 2 > /dev/null 2>&1; echo "14i rc=$?"
timeout 600 $NCU -k regex:fft_rows -s 2 -c 1 -o $D/rows_2p5_split -f python scripts/sweep.py --sizes 5 --layouts split --steps 1 --warmup 2 > /dev/null 2>&1; echo "5 rc=$?"
timeout 600 $NCU -k regex:fft_group -s 2 -c 2 -o $D/group512_2p18_split -f python scripts/sweep.py --sizes 18 --layouts split --steps 1 --warmup 1 > /dev/null 2>&1; echo "18 rc=$?"
timeout 900 $NCU -k regex:fft_group_plane -s 2 -c 2 -o $D/plane4096_2p24_il -f python scripts/sweep.py --sizes 24 --layouts interleaved --batch 8 --steps 1 --warmup 1 > /dev/null 2>&1; echo "24 rc=$?"
ls -la $D
python profiles/summarize.py $D r2ae > $D/summarize.log 2>&1; echo "summarize rc=$?"
mkdir -p $D/txt && cp profiles/r2ae_* $D/txt/ 2>/dev/null; cp profiles/ncu_summary.json $D/txt/ 2>/dev/null
rm -f $D/*.ncu-rep
ls $D/txt
