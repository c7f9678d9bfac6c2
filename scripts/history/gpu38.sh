set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g38_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 300 python scripts/prof_parts.py > $OUT/g38_parts.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q --timeout=300 -k "threshold or solver" > $OUT/g38_pytest.log 2>&1; echo "rc=$?" >> $OUT/g38_pytest.log
echo done
