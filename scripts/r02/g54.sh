#!/bin/bash
# bounded select v2 (one vote per epilogue chunk; select kernel with one round trip of loads and
# vectorised ranks): bounded tests; config-5 bench on (0.8, 0.7) / off; ncu launch list (on)
OUT=gpurun_out/r02g54; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -rf -s -k "bounded" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
S="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
IHT_BOUNDED=0 timeout 600 $B > $OUT/bench_off.json 2> $OUT/bench_off.err
for bd in 0.8 0.7; do IHT_BOUND=$bd IHT_BOUNDED_STATS=1 timeout 600 $B > $OUT/bench_on$bd.json 2> $OUT/bench_on$bd.err; done
IHT_BOUND=0.8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $OUT/launches_on.csv $S > $OUT/ncu_on.log 2>&1
