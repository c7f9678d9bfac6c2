#!/bin/bash
OUT=gpurun_out/r02g05; mkdir -p $OUT
timeout 600 python scripts/r02/fused_tl.py 2 > $OUT/tl.log 2>&1; echo "rc=$?" >> $OUT/tl.log
