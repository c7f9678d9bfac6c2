#!/bin/bash
# One GPU session: tests, bench, launch list and one ncu --set full capture of the adjoint.
# Usage (under gpurun): bash scripts/gpu_round.sh <tag> [bench args...]
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
python bench.py "$@" > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?" >> $OUT/${TAG}_bench.err
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $*"
$SHORT > $OUT/${TAG}_short.json 2> $OUT/${TAG}_short.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/${TAG}_launches.csv $SHORT > $OUT/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?" >> $OUT/${TAG}_short.err
$SHORT > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adjoint_mma -s 3 -c 1 -o $OUT/${TAG}_adjoint $SHORT > $OUT/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> $OUT/${TAG}_short.err
