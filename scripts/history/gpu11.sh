set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g11_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q > $OUT/g11_pytest.log 2>&1; echo "rc=$?" >> $OUT/g11_pytest.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g11_b5.json 2> $OUT/g11_b5.err
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g11_b2.json 2> $OUT/g11_b2.err
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/g11_launch_b5.csv python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
