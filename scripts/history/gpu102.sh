set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g102_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:forward --launch-skip 150 -c 5 --csv \
    --log-file $OUT/g102_fwd_c4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:forward --launch-skip 600 -c 5 --csv \
    --log-file $OUT/g102_fwd_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:forward --launch-skip 600 -c 5 --csv \
    --log-file $OUT/g102_fwd_c2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
