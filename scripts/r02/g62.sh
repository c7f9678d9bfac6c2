#!/bin/bash
# checked build (IHT_LIB=checked: device bounds checks + bounded waits) over the batched, bounded
# select and report tests; config 5 bench (regular build) after the limb refactor
OUT=gpurun_out/r02g62; mkdir -p $OUT
IHT_LIB=checked timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_report.py -m gpu -q -x -rf -p no:cacheprovider > $OUT/pytest_checked.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_checked.log
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c5.json 2> $OUT/c5.err
IHT_BOUNDED=0 timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c5_off.json 2> $OUT/c5_off.err
