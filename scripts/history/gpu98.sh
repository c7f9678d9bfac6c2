set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g98_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/g98_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g98_tests.log
for c in 2 3 5 1; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g98_bench_c$c.json 2> $OUT/g98_bench_c$c.err; done
echo done
