#!/bin/bash
# ncu evidence for one round: launch lists (gpu__time_duration, --clock-control none) of a
# short config-4 and config-5 bench, and one --set full capture of each dominant kernel.
# Each ncu command runs only after the same command exited 0 without ncu (recipe).
TAG=${1:-prof}
OUT=gpurun_out
mkdir -p $OUT
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
C5="python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $C4 > $OUT/${TAG}_c4_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/${TAG}_c4_launches.csv $C4 > /dev/null 2>&1
echo "c4 launches rc=$?" >> $OUT/${TAG}_rc.txt
timeout 900 $C4 > /dev/null 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:adjoint_mma -s 3 -c 1 -o $OUT/${TAG}_c4_adjoint $C4 > $OUT/${TAG}_c4_full.log 2>&1
echo "c4 full rc=$?" >> $OUT/${TAG}_rc.txt
timeout 900 $C5 > $OUT/${TAG}_c5_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/${TAG}_c5_launches.csv $C5 > /dev/null 2>&1
echo "c5 launches rc=$?" >> $OUT/${TAG}_rc.txt
timeout 900 $C5 > /dev/null 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:adjoint_batched -s 3 -c 1 -o $OUT/${TAG}_c5_adjoint $C5 > $OUT/${TAG}_c5_full.log 2>&1
echo "c5 full rc=$?" >> $OUT/${TAG}_rc.txt
