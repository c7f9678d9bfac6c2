#!/bin/bash
OUT=gpurun_out/r02g12; mkdir -p $OUT
TL_CTAS=0 timeout 600 python scripts/r02/fused_tl.py 1 2 3 >> $OUT/tl.log 2>&1
timeout 600 python scripts/r02/fused_check.py > $OUT/fused_check.log 2>&1; echo "rc=$?" >> $OUT/fused_check.log
