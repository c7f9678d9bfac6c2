#!/bin/bash
OUT=gpurun_out/r02g22; mkdir -p $OUT
python scripts/r02/fused_one.py 2 20 > $OUT/run.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fused_iht -c 1 -o $OUT/fused_c2 python scripts/r02/fused_one.py 2 20 > $OUT/ncu.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu.log
