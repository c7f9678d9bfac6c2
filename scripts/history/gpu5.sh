set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g5_build.log 2>&1
for pr in 0 1 2 7; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 300 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g5_probe.log
for b in 4 8; do echo "$(timeout 300 python scripts/prof_batched.py 64 $b 2>&1 | tail -1)"; done >> $OUT/g5_probe.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $OUT/g5_launch0.csv python scripts/prof_batched.py > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_batched.py -x -q > $OUT/g5_pytest_batched.log 2>&1; echo "rc=$?" >> $OUT/g5_pytest_batched.log
echo done
