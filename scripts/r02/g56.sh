#!/bin/bash
# bounded select with the full select inside the same CTA (no cluster-kernel launch): batched +
# config-5 trajectory tests; config-5 bench on / off; launch list
OUT=gpurun_out/r02g56; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_trajectory.py -m gpu -q -x -rf -s -k "batched or config5" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
S="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
IHT_BOUNDED=0 timeout 600 $B > $OUT/bench_off.json 2> $OUT/bench_off.err
IHT_BOUNDED_STATS=1 timeout 600 $B > $OUT/bench_on.json 2> $OUT/bench_on.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $OUT/launches_on.csv $S > $OUT/ncu_on.log 2>&1
