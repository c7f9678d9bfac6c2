#!/bin/bash
# batched GEMM converters: every tile-step of a K-block converted before the stage wait (probe 512)
# against the first only; batched tests under the probe; config 5 A/B x2 interleaved
OUT=gpurun_out/r02g63; mkdir -p $OUT
IHT_BATCHED_PROBE=512 timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -rf -p no:cacheprovider > $OUT/pytest_p512.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_p512.log
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $B > $OUT/c5_base_$rep.json 2> $OUT/c5_base_$rep.err
  IHT_BATCHED_PROBE=512 timeout 600 $B > $OUT/c5_p512_$rep.json 2> $OUT/c5_p512_$rep.err
done
for bits in 4; do
  timeout 600 python bench.py --config 5 --bits $bits --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c5_b${bits}_base.json 2> $OUT/c5_b${bits}_base.err
  IHT_BATCHED_PROBE=512 timeout 600 python bench.py --config 5 --bits $bits --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c5_b${bits}_p512.json 2> $OUT/c5_b${bits}_p512.err
done
