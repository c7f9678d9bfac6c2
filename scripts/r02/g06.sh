#!/bin/bash
OUT=gpurun_out/r02g06; mkdir -p $OUT
for pr in 0 1 2 4 7; do echo "probe $pr" >> $OUT/tl.log; IHT_FUSED_PROBE=$pr timeout 300 python scripts/r02/fused_tl.py 2 >> $OUT/tl.log 2>&1; done
