set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g84_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -m gpu -x -q --timeout 300 -k "forward or solver or teacher" > $OUT/g84_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g84_tests.log
for c in 5 2 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g84_bench_c$c.json 2> $OUT/g84_bench_c$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:forward --launch-skip 600 -c 5 --csv \
    --log-file $OUT/g84_fwd_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
