set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g15_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 300 python scripts/prof_parts.py > $OUT/g15_parts.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_adaptive.py -x -q --timeout=300 > $OUT/g15_pytest_ad.log 2>&1; echo "rc=$?" >> $OUT/g15_pytest_ad.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q --timeout=240 > $OUT/g15_pytest.log 2>&1; echo "rc=$?" >> $OUT/g15_pytest.log
echo done
