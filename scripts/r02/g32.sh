#!/bin/bash
# config-5 batched adjoint: probe matrix and per-CTA timeline
OUT=gpurun_out/r02g32; mkdir -p $OUT
for pr in 0 32 64 16 2 8 1 4; do echo "== probe $pr" >> $OUT/batched.log; IHT_BATCHED_PROBE=$pr timeout 120 python scripts/prof_batched.py 64 2 >> $OUT/batched.log 2>&1; done
