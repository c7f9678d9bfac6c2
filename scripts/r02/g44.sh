#!/bin/bash
# adjoint tail balance: N = 262144 (16384 tasks = 27.7 per warp) vs N = 255744 (15984 tasks =
# exactly 27 per warp at 2 K-ranges x 74 CTAs x 8 warps) vs 254592 (26.9)
OUT=gpurun_out/r02g44; mkdir -p $OUT
for n in 262144 255744 254592 246272; do timeout 120 python scripts/r02/adj_c4.py 4 $n >> $OUT/adj.log 2>&1; done
for n in 262144 255744; do timeout 120 python scripts/r02/adj_c4.py 2 $n >> $OUT/adj.log 2>&1; done
