set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g41_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --timeout=900 -k "config5 or config3" > $OUT/g41_pytest.log 2>&1; echo "rc=$?" >> $OUT/g41_pytest.log
echo done
