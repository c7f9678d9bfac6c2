set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g46_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 2 3; do
  timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --launch-skip 3000 -c 60 --csv \
    --log-file $OUT/g46_launch_c$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g46_ncu_c$c.log 2>&1
done
echo done
