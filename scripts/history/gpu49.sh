set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g49_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/g49_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g49_tests.log
for c in 2 3; do for pr in 0 3; do
  IHT_THR_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_cluster --launch-skip 600 -c 5 --csv \
    --log-file $OUT/g49_thr_c${c}_p$pr.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done; done
for c in 2 3 5; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/g49_bench_c$c.json 2> $OUT/g49_bench_c$c.err; done
echo done
