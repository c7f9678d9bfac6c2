set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g48_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 2 3; do for pr in 0 3 4 5 6; do
  IHT_THR_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_cluster --launch-skip 600 -c 5 --csv \
    --log-file $OUT/g48_thr_c${c}_p$pr.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done; done
echo done
