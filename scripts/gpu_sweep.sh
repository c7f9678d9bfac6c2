#!/bin/bash
# Bench sweep under gpurun: configs 1-5, bit sweep on configs 4 and 5, FFMA baseline,
# adaptive step on config 2, reference arm.
TAG=${1:-sweep}
OUT=gpurun_out
mkdir -p $OUT
for args in "--config 4" "--config 4 --bits 2 --no-cpu-baseline" "--config 4 --bits 8 --no-cpu-baseline" \
            "--config 5" "--config 5 --bits 4 --no-cpu-baseline" "--config 5 --bits 8 --no-cpu-baseline" \
            "--config 2" "--config 3" "--config 1" "--config 2 --adaptive --no-cpu-baseline" \
            "--config 2 --fresh --no-cpu-baseline" \
            "--config 4 --variant 1 --no-cpu-baseline --no-e2e --steps 3"; do
  name=$(echo "$args" | tr -d ' -' )
  timeout 900 python bench.py $args > $OUT/${TAG}_${name}.json 2> $OUT/${TAG}_${name}.err
  echo "$args rc=$?" >> $OUT/${TAG}_rc.txt
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_reference.json 2> $OUT/${TAG}_reference.err
echo "reference rc=$?" >> $OUT/${TAG}_rc.txt
