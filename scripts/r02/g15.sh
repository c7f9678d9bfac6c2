#!/bin/bash
# NEXT-4 tensor-core rate microbenchmark + compute-sanitizer runs
OUT=gpurun_out/r02g15; mkdir -p $OUT
for c in i8 i8n256 bf16 e4m3 e2m1 e2m1n128 mxf4 imma8 imma16 imma32; do timeout 60 scripts/microbench/next4_bench $c >> $OUT/next4.jsonl 2>&1; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv >> $OUT/next4.jsonl 2>&1
for tool in memcheck racecheck synccheck; do
  for w in forward adjoint threshold batched fused solver; do
    echo "== $tool $w" >> $OUT/sanitizer_$tool.log
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/r02/sanitize_cases.py $w >> $OUT/sanitizer_$tool.log 2>&1
    echo "rc=$?" >> $OUT/sanitizer_$tool.log
  done
done
