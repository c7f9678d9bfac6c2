set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g87_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q --timeout 300 > $OUT/g87_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g87_tests.log
for a in "--config 3" "--config 2" "--config 4" "--config 1"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/g87_$n.json 2> $OUT/g87_$n.err
done
echo done
