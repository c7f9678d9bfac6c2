set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g10_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q > $OUT/g10_pytest.log 2>&1; echo "rc=$?" >> $OUT/g10_pytest.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g10_b5.json 2> $OUT/g10_b5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:forward_kernel -s 10 -c 1 -o $OUT/g10_fwd5 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/g10_ncu5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:thr_cluster -s 10 -c 1 -o $OUT/g10_thr5 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/g10_ncu5t.log 2>&1
echo done
