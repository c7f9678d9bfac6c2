set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g62_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "adjoint or solver" > $OUT/g62_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g62_tests.log
for c in 2 3; do for rg in 2 3; do
IHT_ADJ_RING=$rg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:adjoint_mma --launch-skip 300 -c 3 --csv \
    --log-file $OUT/g62_adj_c${c}_r$rg.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done; done
for c in 2 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g62_bench_c$c.json 2> $OUT/g62_bench_c$c.err; done
echo done
