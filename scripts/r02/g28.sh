#!/bin/bash
# k-step microbenchmark; ncu --set full of the fused solver kernel at config 3 (source-level stalls)
OUT=gpurun_out/r02g28; mkdir -p $OUT
timeout 120 ./scripts/microbench/kstep_bench > $OUT/kstep.jsonl 2>&1
timeout 300 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/c3.json 2> $OUT/c3.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_iht -c 1 -o $OUT/c3_fused python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c3.log 2>&1
