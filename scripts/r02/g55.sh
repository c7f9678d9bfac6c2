#!/bin/bash
# NOTE (read after the run): without the fallback the first iteration leaves x = 0, so every later iteration is
# degenerate (empty support: no forward loads, no candidates) -- the nofb / both numbers are not a cost measurement
# config 5, in-graph cost of the pieces around the GEMM (timing only): full / no fallback cluster
# launch (IHT_BOUNDED_NOFB) / no limb kernel (probe 256, stale image) / both
OUT=gpurun_out/r02g55; mkdir -p $OUT
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > $OUT/full.json 2> $OUT/full.err
IHT_BOUNDED_NOFB=1 timeout 600 $B > $OUT/nofb.json 2> $OUT/nofb.err
IHT_BATCHED_PROBE=256 timeout 600 $B > $OUT/nolimbs.json 2> $OUT/nolimbs.err
IHT_BOUNDED_NOFB=1 IHT_BATCHED_PROBE=256 timeout 600 $B > $OUT/both.json 2> $OUT/both.err
