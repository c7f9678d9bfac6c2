#!/bin/bash
# ncu --set full of the fused kernel (config 2) and of the k-step microbenchmark: where do the A phase's cycles go
OUT=gpurun_out/r02g37; mkdir -p $OUT
timeout 300 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/c2.json 2> $OUT/c2.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_iht -c 1 -o $OUT/c2_fused python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c2.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:kstep -c 2 -o $OUT/kstep ./scripts/microbench/kstep_bench > $OUT/ncu_kstep.log 2>&1
