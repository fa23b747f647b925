#!/bin/bash
# Profile captures used for profiles/ (run under gpurun, 1 GPU).  Each command
# is run once plainly first (must exit 0), then under ncu.
set -e
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
NET="python bench.py --ns 4,16 --steps 1 --warmup 1 --no-e2e --no-cpu"
SEG="python tools/workloads.py --which cfg4 --reps 1"
$NET > $OUT/plain_net.log 2>&1
$SEG > $OUT/plain_seg.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:net_(sort|direct)_kernel" -s 0 -c 8 -o $OUT/net -f $NET > $OUT/ncu_net.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 1 -c 1 -o $OUT/seg -f $SEG > $OUT/ncu_seg.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/plain_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launch.log 2>&1
echo done
