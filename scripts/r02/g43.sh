#!/bin/bash
# config-4 experiments: forward address pattern (tiled vs column strips) x words per CTA;
# adjoint K-range / ring depth; bulk-copy stream rate vs bytes in flight
OUT=gpurun_out/r02g43; mkdir -p $OUT
for st in 0 1; do for w in 8 16 32; do IHT_FWD_STRIPS=$st IHT_FWD_WORDS=$w timeout 120 python scripts/r02/fwd_layout.py strips=$st words=$w >> $OUT/fwd.log 2>&1; done; done
for b in 4 2; do
timeout 120 python scripts/r02/adj_c4.py $b >> $OUT/adj.log 2>&1
IHT_ADJ_RING=5 IHT_ADJ_KR=16384 timeout 120 python scripts/r02/adj_c4.py $b >> $OUT/adj.log 2>&1
IHT_ADJ_KR=16384 timeout 120 python scripts/r02/adj_c4.py $b >> $OUT/adj.log 2>&1
done
timeout 300 ./scripts/microbench/bulk_bench > $OUT/bulk.log 2>&1
