set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g63_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_fullsize.py -m gpu -x -q --timeout 300 > $OUT/g63_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g63_tests.log
for sp in 0 1; do echo "split $sp: $(IHT_BATCHED_SPLIT=$sp timeout 120 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g63_prof.log
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/g63_bench_c5.json 2> $OUT/g63_bench_c5.err
echo done
