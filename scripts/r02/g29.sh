#!/bin/bash
# fused A-phase software pipelining + bounded candidates; fresh-adjoint grid sizing
OUT=gpurun_out/r02g29; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "free_running or fused_bounded or teacher" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
TL_CTAS=0 timeout 300 python scripts/r02/fused_tl.py 2 3 > $OUT/fused_tl.log 2>&1
for c in 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 600 python -m pytest tests/test_gpu_trajectory.py tests/test_gpu_fresh.py -m gpu -q -x -rf -p no:cacheprovider > $OUT/pytest2.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest2.log
timeout 900 python bench.py --fresh --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_c4_fresh.json 2> $OUT/bench_c4_fresh.err
timeout 600 python bench.py --config 2 --fresh --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_c2_fresh.json 2> $OUT/bench_c2_fresh.err
