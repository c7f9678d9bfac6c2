set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g56_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 1 2 3 5; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/g56_bench_c$c.json 2> $OUT/g56_bench_c$c.err; done
echo done
