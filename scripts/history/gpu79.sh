set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g79_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fresh.py -m gpu -x -q --timeout 300 > $OUT/g79_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g79_tests.log
for a in "--config 3" "--config 2" "--config 4 --bits 2" "--config 4"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline > $OUT/g79_$n.json 2> $OUT/g79_$n.err
done
echo done
