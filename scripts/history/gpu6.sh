set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g6_build.log 2>&1
for pr in 0 8 9 10 12 13; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 300 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g6_probe.log
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/g6_b5short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $OUT/g6_launch_b5.csv python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
