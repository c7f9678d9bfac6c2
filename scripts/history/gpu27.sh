set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g27_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for cl in 1 4; do for pr in 0 1 2 3; do echo "CL $cl probe $pr: $(IHT_THR_CL=$cl IHT_THR_PROBE=$pr timeout 120 python scripts/prof_parts.py c2 2>&1 | tail -1)"; done; done > $OUT/g27_probe.log
timeout 600 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/g27_launch_c2.csv python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
