set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g13_build.log 2>&1
timeout 600 python scripts/prof_parts.py > $OUT/g13_parts.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q > $OUT/g13_pytest.log 2>&1; echo "rc=$?" >> $OUT/g13_pytest.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g13_b5.json 2> $OUT/g13_b5.err
echo done
