mkdir -p gpurun_out/s5f
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s5f/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5f/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/s5f/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s5f/bench_c4.json 2> gpurun_out/s5f/bench_c4.err
timeout 600 python bench.py --config 6 > gpurun_out/s5f/bench_c6.json 2> gpurun_out/s5f/bench_c6.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s5f/ref_c4.json 2> gpurun_out/s5f/ref_c4.err
