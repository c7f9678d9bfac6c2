#!/bin/bash
# forward_split_kernel (config 4: row blocks x 2 column groups, 16-byte loads) vs forward_kernel;
# forward / solver parity; config-4 bench + launch list
OUT=gpurun_out/r02g50; mkdir -p $OUT
for sp in 1 0; do IHT_FWD_SPLIT=$sp timeout 120 python scripts/r02/fwd_layout.py split=$sp >> $OUT/fwd.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -rf -k "forward or free_running or teacher or config4 or gridsel" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_c4.csv $SHORT > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
