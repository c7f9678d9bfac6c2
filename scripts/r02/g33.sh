#!/bin/bash
# config-5 batched adjoint: combined probes (is the limb-image L2 stream the common floor?)
OUT=gpurun_out/r02g33; mkdir -p $OUT
for pr in 0 1 9 3 65 17 25 27 11; do echo "== probe $pr" >> $OUT/batched.log; IHT_BATCHED_PROBE=$pr timeout 120 python scripts/prof_batched.py 64 2 >> $OUT/batched.log 2>&1; done
