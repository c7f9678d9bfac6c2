set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g32_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for pr in 0 9 2; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 120 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g32_probe.log
for b in 4 8; do echo "$(timeout 120 python scripts/prof_batched.py 64 $b 2>&1 | tail -1)"; done >> $OUT/g32_probe.log
IHT_BATCHED_PROBE=32 timeout 120 python scripts/prof_batched.py > $OUT/g32_tl.log 2>&1
IHT_BATCHED_PROBE=41 timeout 120 python scripts/prof_batched.py > $OUT/g32_tl41.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -x -q --timeout=400 > $OUT/g32_pytest.log 2>&1; echo "rc=$?" >> $OUT/g32_pytest.log
echo done
