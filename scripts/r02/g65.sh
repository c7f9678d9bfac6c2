#!/bin/bash
# fused solver: bounded candidates decided by their count (>= s keys >= the bound: exact), the
# histogram built only when the bound misses; fused / trajectory tests; configs 2/3 at bounds
# 0.9 / 0.7 / 0.5; phase timelines
OUT=gpurun_out/r02g65; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py -m gpu -q -x -rf -k "fused or free_running or config2 or config3" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for c in 2 3; do
  for bd in 0.9 0.7 0.5; do
    IHT_FUSED_BOUND=$bd timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c${c}_b$bd.json 2> $OUT/c${c}_b$bd.err
  done
  IHT_FUSED_NOBOUND=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c${c}_nobound.json 2> $OUT/c${c}_nobound.err
done
TL_CTAS=0 timeout 300 python scripts/r02/fused_tl.py 2 3 > $OUT/tl.log 2>&1
