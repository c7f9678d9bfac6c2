set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g36_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 300 python scripts/prof_parts.py > $OUT/g36_parts.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=600 > $OUT/g36_pytest.log 2>&1; echo "rc=$?" >> $OUT/g36_pytest.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/g36_bench.json 2> $OUT/g36_bench.err
timeout 900 python bench.py --config 5 --no-cpu-baseline > $OUT/g36_bench5.json 2> $OUT/g36_bench5.err
echo done
