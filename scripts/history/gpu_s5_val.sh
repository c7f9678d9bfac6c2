set -x
mkdir -p gpurun_out/s5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s5/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/s5/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s5/bench_c4.json 2> gpurun_out/s5/bench_c4.err
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/s5/bench_c5.json 2> gpurun_out/s5/bench_c5.err
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/s5/bench_c2.json 2> gpurun_out/s5/bench_c2.err
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/s5/bench_c3.json 2> gpurun_out/s5/bench_c3.err
