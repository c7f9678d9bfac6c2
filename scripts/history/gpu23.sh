set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g23_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 120 python scripts/prof_parts.py > $OUT/g23_parts.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_adaptive.py -x -q --timeout=240 > $OUT/g23_pytest.log 2>&1; echo "rc=$?" >> $OUT/g23_pytest.log
echo done
