#!/bin/bash
# fused S2: each CTA's first 8 candidate slots requested with the counts in S1 (one L2 round
# trip fewer on the bounded path); fused / trajectory / free-running tests; configs 2/3 benches
OUT=gpurun_out/r02g68; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py tests/test_gpu_report.py -m gpu -q -x -rf -k "fused or free_running or config2 or config3 or report" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for c in 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c$c.json 2> $OUT/c$c.err; done
TL_CTAS=0 timeout 300 python scripts/r02/fused_tl.py 2 3 > $OUT/tl.log 2>&1
