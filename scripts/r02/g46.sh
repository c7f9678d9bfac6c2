#!/bin/bash
# onepass H_s (cooperative, grid barrier) vs T1-T3; pipelined forward; threshold + solver tests; config-4 bench
OUT=gpurun_out/r02g46; mkdir -p $OUT
timeout 300 python scripts/r02/c4_thr.py >> $OUT/parts.log 2>&1
IHT_THR_ONEPASS=0 timeout 300 python scripts/r02/c4_thr.py >> $OUT/parts.log 2>&1
for w in 8 16 32; do IHT_FWD_WORDS=$w timeout 120 python scripts/r02/fwd_layout.py words=$w >> $OUT/parts.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "threshold or gridsel or forward" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_c4.csv $SHORT > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
