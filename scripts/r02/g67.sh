#!/bin/bash
# ncu --set full captures, config 5 with the bounded select: the tcgen05 GEMM (epilogue lists)
# and thr_bounded_select; config 2 fused kernel (count criterion)
OUT=gpurun_out/r02g67; mkdir -p $OUT
S5="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adjoint_batched_kernel -s 20 -c 1 -o $OUT/c5_gemm $S5 > $OUT/ncu_gemm.log 2>&1; echo "rc=$?" >> $OUT/ncu_gemm.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:thr_bounded_select -s 20 -c 1 -o $OUT/c5_select $S5 > $OUT/ncu_select.log 2>&1; echo "rc=$?" >> $OUT/ncu_select.log
S2="python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_iht_kernel -s 1 -c 1 -o $OUT/c2_fused $S2 > $OUT/ncu_fused.log 2>&1; echo "rc=$?" >> $OUT/ncu_fused.log
