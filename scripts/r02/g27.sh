#!/bin/bash
# phase timelines of the fused solver (configs 2, 3), H_s / forward parts at config 4,
# NEXT-2 fresh copies at config 4 (bench) + one ncu --set full capture of adjoint_fresh_kernel
OUT=gpurun_out/r02g27; mkdir -p $OUT
TL_CTAS=0,-1 timeout 300 python scripts/r02/fused_tl.py 2 3 > $OUT/fused_tl.log 2>&1
for w in 16 32; do IHT_FWD_WORDS=$w timeout 300 python scripts/r02/c4_parts.py forward >> $OUT/parts.log 2>&1; done
timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
timeout 900 python bench.py --fresh --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_c4_fresh.json 2> $OUT/bench_c4_fresh.err
timeout 600 python bench.py --config 2 --fresh --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_c2_fresh.json 2> $OUT/bench_c2_fresh.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adjoint_fresh -s 3 -c 1 -o $OUT/c2_fresh_adjoint python bench.py --config 2 --fresh --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_fresh.log 2>&1
