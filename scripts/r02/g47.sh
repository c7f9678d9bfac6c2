#!/bin/bash
# adjoint prologue (whole lane chunks per thread, 16 float4 in flight) + probes; adjoint parity tests;
# ncu --set full of the config-4 forward and of thr_onepass
OUT=gpurun_out/r02g47; mkdir -p $OUT
for pr in 0 1; do IHT_ADJ_PROBE=$pr timeout 120 python scripts/r02/adj_c4.py 4 >> $OUT/adj.log 2>&1; echo "probe $pr" >> $OUT/adj.log; done
timeout 120 python scripts/r02/adj_c4.py 2 >> $OUT/adj.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -rf -k "adjoint or free_running or teacher or config4" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:forward_kernel -s 5 -c 1 -o $OUT/fwd_c4 $SHORT > $OUT/ncu_fwd.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_fwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:thr_onepass -s 5 -c 1 -o $OUT/onepass_c4 $SHORT > $OUT/ncu_op.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_op.log
