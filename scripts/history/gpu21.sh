set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g21_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for pr in 0 25; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 120 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g21_probe.log
for b in 4 8; do echo "$(timeout 120 python scripts/prof_batched.py 64 $b 2>&1 | tail -1)"; done >> $OUT/g21_probe.log
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q --timeout=240 > $OUT/g21_pytest.log 2>&1; echo "rc=$?" >> $OUT/g21_pytest.log
echo done
