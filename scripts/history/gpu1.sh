set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g1_build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/g1_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/g1_pytest.log
timeout 300 python scripts/dev_batched.py > $OUT/g1_dev_batched.log 2>&1
timeout 300 python scripts/prof_batched.py > $OUT/g1_prof_batched.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adjoint_batched -s 3 -c 1 -o $OUT/g1_batched python scripts/prof_batched.py > $OUT/g1_ncu_batched.log 2>&1
echo done
