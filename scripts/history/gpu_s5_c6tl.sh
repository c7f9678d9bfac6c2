mkdir -p gpurun_out/s5
for b in 0.5 0.7 0.85; do IHT_FUSED_BOUND=$b timeout 300 python bench.py --config 6 --no-cpu-baseline --no-e2e > gpurun_out/s5/c6_bound$b.json 2>/dev/null; done
IHT_FUSED_NOBOUND=1 timeout 300 python bench.py --config 6 --no-cpu-baseline --no-e2e > gpurun_out/s5/c6_nobound.json 2>/dev/null
IHT_FUSED_TL=0 timeout 300 python bench.py --config 6 --steps 2 --no-cpu-baseline --no-e2e > gpurun_out/s5/c6_tl.json 2> gpurun_out/s5/c6_tl.err
IHT_FUSED_TL=0 timeout 300 python bench.py --config 3 --steps 2 --no-cpu-baseline --no-e2e > gpurun_out/s5/c3_tl.json 2> gpurun_out/s5/c3_tl.err
