set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g95_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "adjoint or solver" > $OUT/g95_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g95_tests.log
for a in "--config 4 --bits 2" "--config 4" "--config 3" "--config 4 --bits 2"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> $OUT/g95_$n.json 2> $OUT/g95_$n.err
done
echo done
