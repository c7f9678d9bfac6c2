set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g99_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
echo "prof: $(timeout 120 python scripts/prof_batched.py 2>&1 | tail -1)" > $OUT/g99_prof.log
echo "prof 4-bit: $(timeout 120 python scripts/prof_batched.py 64 4 2>&1 | tail -1)" >> $OUT/g99_prof.log
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_fullsize.py -m gpu -x -q --timeout 300 > $OUT/g99_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g99_tests.log
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g99_bench_c5.json 2> $OUT/g99_bench_c5.err
echo done
