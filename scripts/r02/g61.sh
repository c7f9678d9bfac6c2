#!/bin/bash
# limb image folded into the batched forward (last CTA per snapshot): batched / bounded / report
# tests; config-5 bench fold on / off (IHT_FOLD_LIMBS=0) / bounded off; launch list
OUT=gpurun_out/r02g61; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_report.py -m gpu -q -x -rf -s -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > $OUT/c5.json 2> $OUT/c5.err
IHT_FOLD_LIMBS=0 timeout 600 $B > $OUT/c5_nofold.json 2> $OUT/c5_nofold.err
IHT_BOUNDED=0 timeout 600 $B > $OUT/c5_off.json 2> $OUT/c5_off.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $OUT/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c5.log 2>&1
