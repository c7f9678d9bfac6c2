set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g25_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
IHT_BATCHED_PROBE=32 timeout 120 python scripts/prof_batched.py > $OUT/g25_tl0.log 2>&1
IHT_BATCHED_PROBE=41 timeout 120 python scripts/prof_batched.py > $OUT/g25_tl9.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fresh.py tests/test_gpu_radio.py -x -q --timeout=400 > $OUT/g25_pytest.log 2>&1; echo "rc=$?" >> $OUT/g25_pytest.log
echo done
