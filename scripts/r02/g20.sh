#!/bin/bash
OUT=gpurun_out/r02g20; mkdir -p $OUT
for pr in 0 1 8 9; do echo "probe $pr" >> $OUT/tl.log; IHT_FUSED_PROBE=$pr TL_CTAS=0 timeout 600 python scripts/r02/fused_tl.py 2 3 >> $OUT/tl.log 2>&1; done
