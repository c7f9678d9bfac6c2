#!/bin/bash
# config-5 GEMM: one accumulator with early release + three A/B stages at 2 bits
OUT=gpurun_out/r02g41; mkdir -p $OUT
for pr in 0 32; do echo "== probe $pr" >> $OUT/batched.log; IHT_BATCHED_PROBE=$pr timeout 120 python scripts/prof_batched.py 64 2 >> $OUT/batched.log 2>&1; done
for b in 4 8; do echo "== bits $b" >> $OUT/batched.log; timeout 120 python scripts/prof_batched.py 64 $b >> $OUT/batched.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_fullsize.py -m gpu -q -x -rf -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
