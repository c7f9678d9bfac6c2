#!/bin/bash
OUT=gpurun_out/r02g10; mkdir -p $OUT
TL_CTAS=-1 timeout 600 python scripts/r02/fused_tl.py 2 3 > $OUT/tl.log 2>&1; echo "rc=$?" >> $OUT/tl.log
