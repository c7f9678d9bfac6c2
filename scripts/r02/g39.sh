#!/bin/bash
# fused A phase block-granular warp assignment
OUT=gpurun_out/r02g39; mkdir -p $OUT
TL_CTAS=0 timeout 300 python scripts/r02/fused_tl.py 2 3 > $OUT/fused_tl.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "free_running or fused_bounded" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for c in 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
