#!/bin/bash
OUT=gpurun_out/r02g13; mkdir -p $OUT
TL_CTAS=0 timeout 600 python scripts/r02/fused_tl.py 1 2 3 >> $OUT/tl.log 2>&1
