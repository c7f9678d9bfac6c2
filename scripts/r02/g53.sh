#!/bin/bash
# bounded select A/B (config 5): off / on (bound 0.8) / on without epilogue lists (probe 128):
# bench ms per step and ncu launch lists of each
OUT=gpurun_out/r02g53; mkdir -p $OUT
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
S="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
IHT_BOUNDED=0 timeout 600 $B > $OUT/bench_off.json 2> $OUT/bench_off.err
IHT_BOUND=0.8 IHT_BOUNDED_STATS=1 timeout 600 $B > $OUT/bench_on.json 2> $OUT/bench_on.err
IHT_BOUND=0.8 IHT_BATCHED_PROBE=128 IHT_BOUNDED_STATS=1 timeout 600 $B > $OUT/bench_noemit.json 2> $OUT/bench_noemit.err
for v in off on noemit; do
  case $v in off) E="IHT_BOUNDED=0";; on) E="IHT_BOUND=0.8";; noemit) E="IHT_BOUND=0.8 IHT_BATCHED_PROBE=128";; esac
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $OUT/launches_$v.csv $S > $OUT/ncu_$v.log 2>&1
done
