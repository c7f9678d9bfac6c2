set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g85_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q --timeout 300 > $OUT/g85_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g85_tests.log
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g85_bench_c5.json 2> $OUT/g85_bench_c5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:limbs --launch-skip 600 -c 5 --csv \
    --log-file $OUT/g85_limbs_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
