set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g14_build.log 2>&1
timeout 300 python scripts/prof_parts.py > $OUT/g14_parts.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q --timeout=240 > $OUT/g14_pytest.log 2>&1; echo "rc=$?" >> $OUT/g14_pytest.log
timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:thr_cluster -s 5 -c 1 -o $OUT/g14_thr python scripts/prof_parts.py c5 > /dev/null 2>&1
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g14_b5.json 2> $OUT/g14_b5.err
echo done
