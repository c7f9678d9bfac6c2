set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g76_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 2 5; do for pr in 1 2 3 4 0; do
IHT_THR_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:thr_cluster --launch-skip 650 -c 3 --csv \
    --log-file $OUT/g76_thr_c${c}_p$pr.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done; done
echo done
