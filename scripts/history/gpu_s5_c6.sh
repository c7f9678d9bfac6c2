set -x
mkdir -p gpurun_out/s5
timeout 900 python -m pytest tests/test_gpu_trajectory.py -k config6 -x -q -s > gpurun_out/s5/c6_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5/c6_tests.log
timeout 600 python bench.py --config 6 > gpurun_out/s5/bench_c6.json 2> gpurun_out/s5/bench_c6.err
timeout 300 python bench.py --config 6 --adaptive --no-cpu-baseline > gpurun_out/s5/bench_c6_adaptive.json 2> gpurun_out/s5/bench_c6_adaptive.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:fused_iht -c 3 --csv --log-file gpurun_out/s5/c6_launches.csv python bench.py --config 6 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/s5/c6_ncu.log 2>&1
