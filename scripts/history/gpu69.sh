set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g69_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 2 3; do for sk in 601 650 750; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_cluster --launch-skip $sk -c 2 --csv \
    --log-file $OUT/g69_thr_c${c}_$sk.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done; done
echo done
