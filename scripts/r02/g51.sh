#!/bin/bash
# bounded select for config 5 (epilogue candidates + thr_bounded_select, cluster kernel only for
# undecided snapshots): bit-identity tests, batched tests, config-5 bench at bounds 0.5 / 0.7 / 0.3
# and with the bounded select off
OUT=gpurun_out/r02g51; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_trajectory.py -m gpu -q -x -rf -s -k "batched or config5" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for bd in 0.5 0.7 0.3; do
  IHT_BOUND=$bd IHT_BOUNDED_STATS=1 timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5_b$bd.json 2> $OUT/bench_c5_b$bd.err
done
IHT_BOUNDED=0 timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5_off.json 2> $OUT/bench_c5_off.err
