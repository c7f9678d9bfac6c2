#!/bin/bash
# MMA order interleaving the accumulators: k-step bench, fused timelines, adjoint configs 3/4
OUT=gpurun_out/r02g31; mkdir -p $OUT
timeout 120 ./scripts/microbench/kstep_bench > $OUT/kstep.jsonl 2>&1
TL_CTAS=0 timeout 300 python scripts/r02/fused_tl.py 2 3 > $OUT/fused_tl.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "adjoint or free_running or fused_bounded" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for c in 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --bits 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4b2.json 2> $OUT/bench_c4b2.err
IHT_THR_MULTI=2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4_cluster.json 2> $OUT/bench_c4_cluster.err
