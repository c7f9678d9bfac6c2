set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g77_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 1000 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/g77_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g77_tests.log
for c in 2 3 5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:thr_cluster --launch-skip 650 -c 3 --csv \
    --log-file $OUT/g77_thr_c$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/g77_bench_c$c.json 2> $OUT/g77_bench_c$c.err
done
echo done
