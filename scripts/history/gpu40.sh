set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g40_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --timeout=600 > $OUT/g40_pytest.log 2>&1; echo "rc=$?" >> $OUT/g40_pytest.log
timeout 300 python scripts/prof_batched.py > $OUT/g40_pb.log 2>&1
echo done
