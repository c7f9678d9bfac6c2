#!/bin/bash
# fused solver variants (bound fraction, no bound, probes) + tcgen05 pair microbenchmark
OUT=gpurun_out/r02g30; mkdir -p $OUT
for v in "IHT_FUSED_BOUND=0.9" "IHT_FUSED_BOUND=0.97" "IHT_FUSED_NOBOUND=1" "IHT_FUSED_NOBOUND=1 IHT_FUSED_PROBE=2" "IHT_FUSED_NOBOUND=1 IHT_FUSED_PROBE=4"; do
  echo "== $v" >> $OUT/fused_tl.log
  env $v TL_CTAS=0 timeout 300 python scripts/r02/fused_tl.py 2 3 >> $OUT/fused_tl.log 2>&1
done
timeout 60 ./scripts/microbench/tc2_bench > $OUT/tc2.jsonl 2>&1; echo "rc=$?" >> $OUT/tc2.jsonl
