#!/bin/bash
# forward decode 2^B + code (one shift + one LOP3 per code); adjoint without the probe-2 branch;
# tests of the forward / fused / batched paths; benches configs 2, 3, 5, 4
OUT=gpurun_out/r02g49; mkdir -p $OUT
for b in 4 2; do timeout 120 python scripts/r02/adj_c4.py $b >> $OUT/adj.log 2>&1; done
IHT_FWD_WORDS=16 timeout 120 python scripts/r02/fwd_layout.py words=16 >> $OUT/adj.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_trajectory.py -m gpu -q -x -rf -k "forward or free_running or teacher or trajectory or fused" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for c in 2 3 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
