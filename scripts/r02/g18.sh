#!/bin/bash
OUT=gpurun_out/r02g18; mkdir -p $OUT
timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
IHT_THR_MULTI=1 timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
