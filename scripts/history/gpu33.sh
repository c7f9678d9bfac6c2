set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g33_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --timeout=600 > $OUT/g33_pytest.log 2>&1; echo "rc=$?" >> $OUT/g33_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/g33_smoke.log 2>&1; echo "rc=$?" >> $OUT/g33_smoke.log
timeout 900 python bench.py > $OUT/g33_bench.json 2> $OUT/g33_bench.err; echo "rc=$?" >> $OUT/g33_bench.err
timeout 600 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/g33_launch_c2.csv python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
