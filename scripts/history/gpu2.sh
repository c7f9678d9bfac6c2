set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g2_build.log 2>&1
timeout 600 python scripts/prof_batched.py > $OUT/g2_prof_batched.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_batched.py -x -q > $OUT/g2_pytest_batched.log 2>&1; echo "rc=$?" >> $OUT/g2_pytest_batched.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/g2_pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/g2_pytest_parity.log
echo done
