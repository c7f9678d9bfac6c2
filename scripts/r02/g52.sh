#!/bin/bash
# bounded select, bound keys from the limb kernel (r02 g51: the epilogue computing them itself
# delayed its first tile, config 5 14.97k -> 11.47k iter/s); tests; config-5 bench at bounds
# 0.7 / 0.8 / 0.9 / 0.5 and off; config-5 ncu launch list at the default
OUT=gpurun_out/r02g52; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -rf -s -k "bounded" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for bd in 0.7 0.8 0.9 0.5; do
  IHT_BOUND=$bd IHT_BOUNDED_STATS=1 timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5_b$bd.json 2> $OUT/bench_c5_b$bd.err
done
IHT_BOUNDED=0 timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5_off.json 2> $OUT/bench_c5_off.err
IHT_BOUND=0.8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
