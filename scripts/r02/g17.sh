#!/bin/bash
OUT=gpurun_out/r02g17; mkdir -p $OUT
for w in 8 16 32; do IHT_FWD_WORDS=$w timeout 300 python scripts/r02/c4_parts.py forward >> $OUT/parts.log 2>&1; done
timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
IHT_THR_TL=1 timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
