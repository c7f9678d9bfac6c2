#!/bin/bash
# adjoint probes at config 4 (1 = no r prologue, 2 = stream only, 3 = both) + onepass H_s tests
OUT=gpurun_out/r02g45; mkdir -p $OUT
for pr in 0 1 2 3; do IHT_ADJ_PROBE=$pr timeout 120 python scripts/r02/adj_c4.py 4 >> $OUT/adj.log 2>&1; echo "probe $pr" >> $OUT/adj.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "threshold or gridsel or free_running" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/r02/c4_thr.py >> $OUT/parts.log 2>&1
IHT_THR_ONEPASS=0 timeout 300 python scripts/r02/c4_thr.py >> $OUT/parts.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
