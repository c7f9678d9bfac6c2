set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g3_build.log 2>&1
for pr in 0 1 2 4 3 5 6 7; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 300 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g3_probe.log
timeout 1200 python -m pytest tests/test_gpu_batched.py -x -q > $OUT/g3_pytest_batched.log 2>&1; echo "rc=$?" >> $OUT/g3_pytest_batched.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > $OUT/g3_bench5.json 2> $OUT/g3_bench5.err
echo done
