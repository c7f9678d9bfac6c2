set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 120 ./scripts/microbench/pipe_bench > $OUT/g17_pipe.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/g17_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 300 python scripts/prof_parts.py > $OUT/g17_parts.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q --timeout=240 -k "threshold or solver or teacher" > $OUT/g17_pytest.log 2>&1; echo "rc=$?" >> $OUT/g17_pytest.log
echo done
