set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g72_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 2 3 5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --launch-skip 2000 -c 40 --csv \
    --log-file $OUT/g72_warm_c$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
echo done
