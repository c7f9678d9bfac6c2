set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g47_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for pr in 1 2 3; do
  IHT_THR_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_cluster --launch-skip 600 -c 10 --csv \
    --log-file $OUT/g47_thr_p$pr.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 400 ncu --set full --import-source on --clock-control none -k regex:thr_cluster --launch-skip 600 -c 1 -o $OUT/g47_thr_c2 -f \
    python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g47_full.log 2>&1
echo done
